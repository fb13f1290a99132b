// jagged.cu — jagged gather / scatter on the device ("fully jagged tensor
// implementation"): shard packing for the data-parallel partition,
// attention truncation's "latest L' rows" slice, padded <-> jagged.
// Row copies are 16-byte vectorised and coalesced along rows; one warp per row.
#include <algorithm>
#include <vector>

#include "internal.h"

namespace uh {
namespace {

constexpr int kSegs = 256;  // segments per launch (kernel-parameter budget)
struct Seg { int32_t src, dst, len; };
struct SegBatch { Seg s[kSegs]; int n; };

// copy `len` rows per segment with VT-wide vectors (uint4: row bytes and both strides multiples of
// 16; uint2: multiples of 8, e.g. int64 timestamps or an odd 8-byte stride)
template <typename VT>
__global__ void __launch_bounds__(256) copy_rows_k(const __grid_constant__ SegBatch b, const uint8_t* __restrict__ x,
                                                   int64_t ldx_bytes, uint8_t* __restrict__ y, int64_t ldy_bytes,
                                                   int64_t row_bytes) {
    const int seg = blockIdx.y;
    if (seg >= b.n) return;
    const Seg s = b.s[seg];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nvec = row_bytes / (int64_t)sizeof(VT);
    if (nvec == 1) {   // narrow rows: one lane per row
        for (int r = (blockIdx.x * 8 + warp) * 32 + lane; r < s.len; r += gridDim.x * 256)
            *reinterpret_cast<VT*>(y + (int64_t)(s.dst + r) * ldy_bytes) =
                *reinterpret_cast<const VT*>(x + (int64_t)(s.src + r) * ldx_bytes);
        return;
    }
    for (int r = blockIdx.x * 8 + warp; r < s.len; r += gridDim.x * 8) {
        const VT* src = reinterpret_cast<const VT*>(x + (int64_t)(s.src + r) * ldx_bytes);
        VT* dst = reinterpret_cast<VT*>(y + (int64_t)(s.dst + r) * ldy_bytes);
        for (int64_t v = lane; v < nvec; v += 32) dst[v] = src[v];
    }
}

template <typename VT>
__global__ void __launch_bounds__(256) zero_rows_k(const __grid_constant__ SegBatch b, uint8_t* __restrict__ y,
                                                   int64_t ldy_bytes, int64_t row_bytes) {
    const int seg = blockIdx.y;
    if (seg >= b.n) return;
    const Seg s = b.s[seg];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nvec = row_bytes / (int64_t)sizeof(VT);
    for (int r = blockIdx.x * 8 + warp; r < s.len; r += gridDim.x * 8) {
        VT* dst = reinterpret_cast<VT*>(y + (int64_t)(s.dst + r) * ldy_bytes);
        for (int64_t v = lane; v < nvec; v += 32) dst[v] = VT{};
    }
}

uh_status run_segments(const std::vector<Seg>& segs, const void* x, int64_t ldx_bytes, void* y, int64_t ldy_bytes,
                       int64_t row_bytes, bool zero, cudaStream_t st) {
    int maxlen = 0;
    for (auto& s : segs) maxlen = std::max(maxlen, s.len);
    if (maxlen == 0) return UH_OK;
    for (size_t i0 = 0; i0 < segs.size(); i0 += kSegs) {
        SegBatch b{};
        b.n = (int)std::min<size_t>(kSegs, segs.size() - i0);
        for (int i = 0; i < b.n; ++i) b.s[i] = segs[i0 + i];
        dim3 grid((unsigned)std::min(64, (maxlen + 7) / 8), (unsigned)b.n);
        // 16-byte vectors only when every row start is 16-byte aligned (row bytes AND both
        // strides): an 8-byte multiple stride puts every odd row 8 bytes off a 16-byte boundary
        const bool v16 = row_bytes % 16 == 0 && ldx_bytes % 16 == 0 && ldy_bytes % 16 == 0;
        if (zero && v16) zero_rows_k<uint4><<<grid, 256, 0, st>>>(b, (uint8_t*)y, ldy_bytes, row_bytes);
        else if (zero) zero_rows_k<uint2><<<grid, 256, 0, st>>>(b, (uint8_t*)y, ldy_bytes, row_bytes);
        else if (v16)
            copy_rows_k<uint4><<<grid, 256, 0, st>>>(b, (const uint8_t*)x, ldx_bytes, (uint8_t*)y, ldy_bytes, row_bytes);
        else
            copy_rows_k<uint2><<<grid, 256, 0, st>>>(b, (const uint8_t*)x, ldx_bytes, (uint8_t*)y, ldy_bytes, row_bytes);
        note_launch();
        UH_CUDA(cudaGetLastError());
    }
    return UH_OK;
}

uh_status check_common(const uh_jagged* j, const void* x, int64_t width, int32_t eb, const void* y) {
    if (!j || !j->host_offsets) return fail(UH_ERR_NULL, "jagged descriptor / host_offsets NULL");
    if (j->num_seqs < 0) return fail(UH_ERR_DOMAIN, "num_seqs < 0");
    if (eb != 1 && eb != 2 && eb != 4 && eb != 8) return fail(UH_ERR_DOMAIN, "elem_bytes must be 1, 2, 4 or 8");
    if (width < 0) return fail(UH_ERR_DOMAIN, "width < 0");
    if ((width * eb) % 8) return fail(UH_ERR_ALIGNMENT, "row bytes must be a multiple of 8");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
        return fail(UH_ERR_ALIGNMENT, "x / y not 16-byte aligned");
    for (int b = 0; b < j->num_seqs; ++b)
        if (j->host_offsets[b + 1] < j->host_offsets[b]) return fail(UH_ERR_DOMAIN, "negative sequence length");
    return UH_OK;
}

uh_status publish_offsets(const std::vector<int32_t>& off, int32_t* host, int32_t* dev, cudaStream_t st) {
    if (host) std::copy(off.begin(), off.end(), host);
    if (dev) UH_CUDA(cudaMemcpyAsync(dev, off.data(), off.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    if (dev) UH_CUDA(cudaStreamSynchronize(st));  // `off` is a local; keep the copy valid
    return UH_OK;
}

}  // namespace
}  // namespace uh

using namespace uh;

extern "C" {

uh_status uh_jagged_gather(const uh_jagged* src, const int32_t* seq_ids, int32_t n, const void* x, int64_t ld_x,
                           int64_t width, int32_t eb, void* y, int32_t* dst_off_host, int32_t* dst_off_dev,
                           void* stream) {
    UH_TRY(check_common(src, x, width, eb, y));
    if (n < 0) return fail(UH_ERR_DOMAIN, "n < 0");
    if (n > 0 && !seq_ids) return fail(UH_ERR_NULL, "seq_ids NULL");
    if (ld_x < width || (ld_x * eb) % 8) return fail(UH_ERR_ALIGNMENT, "ld_x (bytes) must be a multiple of 8");
    std::vector<Seg> segs;
    std::vector<int32_t> off(1, 0);
    for (int i = 0; i < n; ++i) {
        const int id = seq_ids[i];
        if (id < 0 || id >= src->num_seqs) return fail(UH_ERR_DOMAIN, "seq id out of range");
        const int32_t s0 = src->host_offsets[id], L = src->host_offsets[id + 1] - s0;
        segs.push_back(Seg{s0, off.back(), L});
        off.push_back(off.back() + L);
    }
    UH_TRY(run_segments(segs, x, ld_x * eb, y, width * eb, width * eb, false, (cudaStream_t)stream));
    return publish_offsets(off, dst_off_host, dst_off_dev, (cudaStream_t)stream);
}

uh_status uh_jagged_slice_latest(const uh_jagged* src, int32_t l_keep, const void* x, int64_t ld_x, int64_t width,
                                 int32_t eb, void* y, int32_t* dst_off_host, int32_t* dst_off_dev, void* stream) {
    UH_TRY(check_common(src, x, width, eb, y));
    if (l_keep < 0) return fail(UH_ERR_DOMAIN, "l_keep < 0");
    if (ld_x < width || (ld_x * eb) % 8) return fail(UH_ERR_ALIGNMENT, "ld_x (bytes) must be a multiple of 8");
    std::vector<Seg> segs;
    std::vector<int32_t> off(1, 0);
    for (int b = 0; b < src->num_seqs; ++b) {
        const int32_t s0 = src->host_offsets[b], L = src->host_offsets[b + 1] - s0;
        const int32_t keep = std::min(L, l_keep);
        segs.push_back(Seg{s0 + L - keep, off.back(), keep});
        off.push_back(off.back() + keep);
    }
    UH_TRY(run_segments(segs, x, ld_x * eb, y, width * eb, width * eb, false, (cudaStream_t)stream));
    return publish_offsets(off, dst_off_host, dst_off_dev, (cudaStream_t)stream);
}

uh_status uh_jagged_to_padded(const uh_jagged* src, const void* x, int64_t width, int32_t eb, int32_t max_len, void* y,
                              void* stream) {
    UH_TRY(check_common(src, x, width, eb, y));
    std::vector<Seg> segs, pads;
    for (int b = 0; b < src->num_seqs; ++b) {
        const int32_t s0 = src->host_offsets[b], L = src->host_offsets[b + 1] - s0;
        if (L > max_len) return fail(UH_ERR_DIM, "sequence longer than max_len");
        segs.push_back(Seg{s0, b * max_len, L});
        pads.push_back(Seg{0, b * max_len + L, max_len - L});
    }
    UH_TRY(run_segments(pads, nullptr, 0, y, width * eb, width * eb, true, (cudaStream_t)stream));
    return run_segments(segs, x, width * eb, y, width * eb, width * eb, false, (cudaStream_t)stream);
}

uh_status uh_padded_to_jagged(const uh_jagged* dst, const void* y, int64_t width, int32_t eb, int32_t max_len, void* x,
                              void* stream) {
    UH_TRY(check_common(dst, x, width, eb, y));
    std::vector<Seg> segs;
    for (int b = 0; b < dst->num_seqs; ++b) {
        const int32_t s0 = dst->host_offsets[b], L = dst->host_offsets[b + 1] - s0;
        if (L > max_len) return fail(UH_ERR_DIM, "sequence longer than max_len");
        segs.push_back(Seg{b * max_len, s0, L});
    }
    return run_segments(segs, y, width * eb, x, width * eb, width * eb, false, (cudaStream_t)stream);
}

}  // extern "C"
