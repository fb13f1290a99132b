// lbsl.cu — NEXT-3: Load-Balanced Stochastic Length (arXiv 2602.16986 §4.1, P:109-115;
// Algorithm 1) and the device row gather that applies its decisions.
// The per-rank selection is host code (b ~ 32 lengths per step); see
// include/uhstu_lbsl.h for the readings R21-R26 and the counter-based generator.
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/uhstu_lbsl.h"
#include "internal.h"

namespace uh {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
enum : uint64_t { kStreamSL = 0, kStreamPerm = 1, kStreamSubset = 2 };

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// (seed, rank, step, stream, idx) -> uniform in (0, 1); the chain order is the ABI's
inline double ctr_u01(uint64_t seed, int64_t rank, int64_t step, uint64_t stream, uint64_t idx) {
    uint64_t x = seed;
    const uint64_t c[4] = {(uint64_t)rank, (uint64_t)step, stream, idx};
    for (uint64_t v : c) x = mix64(x + kGolden + v);
    return ((double)(x >> 11) + 0.5) * 0x1.0p-53;
}

// R21/R22: StandardSL's keep probability, also SLWeight
inline double keep_prob(int32_t n, int32_t ell) {
    if (n <= ell) return 1.0;
    return ((double)ell * (double)ell) / ((double)n * (double)n);
}

// R21: Knuth's selection sampling; writes tau increasing positions
void subset(int32_t n, int32_t tau, uint64_t seed, int32_t rank, int64_t step, int32_t u, int32_t* idx) {
    int32_t got = 0;
    for (int32_t j = 0; j < n && got < tau; ++j) {
        const double r = ctr_u01(seed, rank, step, kStreamSubset, ((uint64_t)u << 32) | (uint32_t)j);
        if ((double)(n - j) * r < (double)(tau - got)) idx[got++] = j;
    }
}

// device: one warp per row, 16-byte vectors, grid-stride over rows
__global__ void __launch_bounds__(256) gather_rows_k(const int32_t* __restrict__ rows, int64_t n_rows,
                                                      const uint8_t* __restrict__ x, int64_t ldx_bytes,
                                                      uint8_t* __restrict__ y, int64_t ldy_bytes, int64_t vecs) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_rows; i += warps) {
        const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)__ldg(rows + i) * ldx_bytes);
        uint4* dst = reinterpret_cast<uint4*>(y + i * ldy_bytes);
        for (int64_t v = lane; v < vecs; v += 32) dst[v] = __ldg(src + v);
    }
}

}  // namespace
}  // namespace uh

using namespace uh;

extern "C" {

uh_status uh_lbsl_select(const int32_t* lengths, int32_t b, int32_t ell, double gamma, double ell_bar,
                         int32_t steady, uint64_t seed, int32_t rank, int64_t step, int32_t* decision,
                         int32_t* new_len, double* proxy) {
    if (b < 0 || ell < 1 || !(gamma > 0.0) || (steady != 0 && steady != 1))
        return fail(UH_ERR_DOMAIN, "lbsl_select: b >= 0, ell_sl >= 1, gamma > 0, steady in {0,1}");
    if (b > 0 && (!lengths || !decision || !new_len)) return fail(UH_ERR_NULL, "lbsl_select: NULL array");
    if (!proxy) return fail(UH_ERR_NULL, "lbsl_select: proxy_load NULL");
    for (int32_t u = 0; u < b; ++u)
        if (lengths[u] < 0) return fail(UH_ERR_DOMAIN, "lbsl_select: negative length");

    // Alg. 1 line 5 (R22): expected StandardSL load, in index order
    double s5 = 0.0;
    const double ell_g = std::pow((double)ell, gamma);
    for (int32_t u = 0; u < b; ++u) {
        const int32_t n = lengths[u];
        if (n <= ell) {
            s5 += std::pow((double)n, gamma);
        } else {
            const double q = keep_prob(n, ell);
            s5 += q * std::pow((double)n, gamma) + (1.0 - q) * ell_g;
        }
    }
    *proxy = s5;

    if (!steady) {  // line 7: StandardSL on every user
        for (int32_t u = 0; u < b; ++u) {
            const int32_t n = lengths[u];
            const bool trunc = n > ell && ctr_u01(seed, rank, step, kStreamSL, (uint64_t)u) >= keep_prob(n, ell);
            decision[u] = trunc ? UH_LBSL_TRUNCATED : UH_LBSL_KEPT_BY_SL;
        }
    } else {
        // lines 9-11: weights, exponential keys, order (key desc, index asc)
        std::vector<double> key(b), base(b);
        std::vector<int32_t> pi(b);
        double base_sum = 0.0;
        for (int32_t u = 0; u < b; ++u) {
            key[u] = std::log(ctr_u01(seed, rank, step, kStreamPerm, (uint64_t)u)) / keep_prob(lengths[u], ell);
            base[u] = std::pow((double)std::min(lengths[u], ell), gamma);  // R25
            base_sum += base[u];
            pi[u] = u;
        }
        const double budget = ell_bar - base_sum;
        std::sort(pi.begin(), pi.end(), [&](int32_t a, int32_t c) { return key[a] > key[c] || (key[a] == key[c] && a < c); });
        // lines 12-16: greedy fill of the untruncated set U_r
        double s = 0.0;
        for (int32_t u = 0; u < b; ++u) decision[u] = -1;
        for (int32_t k = 0; k < b; ++k) {
            const int32_t u = pi[k];
            const double inc = std::pow((double)lengths[u], gamma) - base[u];
            if (s + inc <= budget) {
                decision[u] = UH_LBSL_UNSAMPLED;
                s = s + inc;
            }
        }
        // lines 17-18 (R26): everyone else is sampled down to l_SL
        for (int32_t u = 0; u < b; ++u)
            if (decision[u] < 0) decision[u] = lengths[u] > ell ? UH_LBSL_TRUNCATED : UH_LBSL_KEPT_BY_SL;
    }
    for (int32_t u = 0; u < b; ++u)
        new_len[u] = decision[u] == UH_LBSL_TRUNCATED ? std::min(lengths[u], ell) : lengths[u];
    return UH_OK;
}

uh_status uh_lbsl_subset(int32_t n, int32_t tau, uint64_t seed, int32_t rank, int64_t step, int32_t u,
                         int32_t* idx) {
    if (n < 0 || tau < 0 || tau > n || u < 0) return fail(UH_ERR_DOMAIN, "lbsl_subset: 0 <= tau <= n, u >= 0");
    if (tau > 0 && !idx) return fail(UH_ERR_NULL, "lbsl_subset: idx NULL");
    subset(n, tau, seed, rank, step, u, idx);
    return UH_OK;
}

uh_status uh_lbsl_rows(const int32_t* off, int32_t b, const int32_t* decision, const int32_t* new_len,
                       uint64_t seed, int32_t rank, int64_t step, int32_t* rows, int32_t* new_off) {
    if (b < 0) return fail(UH_ERR_DOMAIN, "lbsl_rows: b < 0");
    if (!off || !new_off || (b > 0 && (!decision || !new_len))) return fail(UH_ERR_NULL, "lbsl_rows: NULL array");
    int64_t total = 0;
    for (int32_t u = 0; u < b; ++u) {
        const int32_t n = off[u + 1] - off[u];
        if (n < 0) return fail(UH_ERR_DIM, "lbsl_rows: offsets decrease");
        const bool ok = decision[u] == UH_LBSL_TRUNCATED ? (new_len[u] >= 0 && new_len[u] <= n) : new_len[u] == n;
        if (!ok) return fail(UH_ERR_DIM, "lbsl_rows: new_len inconsistent with the decision");
        total += new_len[u];
    }
    if (total > 0 && !rows) return fail(UH_ERR_NULL, "lbsl_rows: rows NULL");
    new_off[0] = 0;
    for (int32_t u = 0; u < b; ++u) {
        const int32_t n = off[u + 1] - off[u], o = new_off[u];
        if (decision[u] == UH_LBSL_TRUNCATED) {
            subset(n, new_len[u], seed, rank, step, u, rows + o);
            for (int32_t j = 0; j < new_len[u]; ++j) rows[o + j] += off[u];
        } else {
            for (int32_t j = 0; j < n; ++j) rows[o + j] = off[u] + j;
        }
        new_off[u + 1] = o + new_len[u];
    }
    return UH_OK;
}

uh_status uh_gather_rows(const int32_t* rows, int64_t n_rows, const void* x, int64_t ld_x, int64_t width, int32_t eb,
                         void* y, int64_t ld_y, void* stream) {
    if (n_rows < 0 || width < 0 || eb <= 0) return fail(UH_ERR_DOMAIN, "gather_rows: n_rows, width >= 0, elem_bytes > 0");
    if (n_rows == 0 || width == 0) return UH_OK;
    if (!rows || !x || !y) return fail(UH_ERR_NULL, "gather_rows: NULL pointer");
    if (ld_x < width || ld_y < width) return fail(UH_ERR_DIM, "gather_rows: ld < width");
    if (((uintptr_t)x | (uintptr_t)y) % 16 || (width * eb) % 16 || (ld_x * eb) % 16 || (ld_y * eb) % 16)
        return fail(UH_ERR_ALIGNMENT, "gather_rows: 16-byte pointers and row bytes");
    const int blocks = (int)std::min<int64_t>((n_rows + 7) / 8, (int64_t)num_sms() * 8);  // 8 warps per block
    gather_rows_k<<<blocks, 256, 0, (cudaStream_t)stream>>>(rows, n_rows, (const uint8_t*)x, ld_x * eb, (uint8_t*)y,
                                                            ld_y * eb, width * eb / 16);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

}  // extern "C"
