// attn_bwd_sm100.cu — placeholder until the tcgen05 backward lands.
#include "attn_common.cuh"
#include "internal.h"
namespace uh {
uh_status attn_bwd_sm100_launch(const AttnArgs& a, const AttnArgs& akv, cudaStream_t st, int64_t T) {
    (void)a; (void)akv; (void)st; (void)T;
    return fail(UH_ERR_UNSUPPORTED, "bf16 attention backward not built yet");
}
}  // namespace uh
