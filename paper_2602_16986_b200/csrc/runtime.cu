// runtime.cu — host runtime pieces of libuhstu: thread-local error detail, the
// driver entry point for TMA descriptors, device properties.
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>
#include <string>

#include "internal.h"
#include "../../include/uhstu_testing.h"

namespace uh {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

uh_status fail(uh_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

uh_status cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return UH_ERR_CUDA;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

uh_status make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                         uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
    auto enc = get_encode();
    if (!enc) return fail(UH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (outer == 0) outer = 1;  // empty tensors are never read; keep the descriptor valid
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(UH_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
    return UH_OK;
}

uh_status make_tmap_u8(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                       uint32_t box_inner, uint32_t box_outer) {
    auto enc = get_encode();
    if (!enc) return fail(UH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (outer == 0) outer = 1;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(UH_ERR_CUDA, "cuTensorMapEncodeTiled (u8) failed (code " + std::to_string((int)r) + ")");
    return UH_OK;
}

uh_status make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer) {
    auto enc = get_encode();
    if (!enc) return fail(UH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (outer == 0) outer = 1;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_elems * 4};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(UH_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed (code " + std::to_string((int)r) + ")");
    return UH_OK;
}

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    static int cache[64] = {0};
    if (dev < 64 && cache[dev]) return cache[dev];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) cache[dev] = n;
    return n;
}

}  // namespace uh

extern "C" const char* uh_last_error(void) { return uh::g_last_error.c_str(); }

extern "C" long long uh_test_launch_count(void) { return uh::launch_count(); }
