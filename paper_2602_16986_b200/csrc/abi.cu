// abi.cu — the exported C ABI of libuhstu (include/uhstu.h): argument
// validation (always before any launch), workspace sizing, the layer
// orchestration of Listing 1 with the rematerialising backward
// (P:187-189), jagged gather/scatter and the host LPT partitioner.
#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>
#include <vector>

#include "gemm_sm100.cuh"  // EPI_* constants
#include "internal.h"

using namespace uh;

namespace {

constexpr int64_t kMaxTokens = INT32_MAX;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
int esize(uh_dtype dt) { return dt == UH_BF16 ? 2 : 4; }
int ld_mult(uh_dtype dt) { return dt == UH_BF16 ? 8 : 4; }

uh_status check_jagged(const uh_jagged* j, bool need_device = true) {
    if (!j) return fail(UH_ERR_NULL, "jagged descriptor is NULL");
    if (j->num_seqs < 0) return fail(UH_ERR_DOMAIN, "num_seqs < 0");
    if (!j->host_offsets) return fail(UH_ERR_NULL, "host_offsets is NULL");
    if (j->host_offsets[0] != 0) return fail(UH_ERR_DIM, "offsets[0] != 0");
    int32_t mx = 0;
    for (int b = 0; b < j->num_seqs; ++b) {
        int32_t L = j->host_offsets[b + 1] - j->host_offsets[b];
        if (L < 0) return fail(UH_ERR_DOMAIN, "negative sequence length at " + std::to_string(b));
        mx = std::max(mx, L);
    }
    if ((int64_t)j->host_offsets[j->num_seqs] != j->total_tokens)
        return fail(UH_ERR_DIM, "offsets[B] != total_tokens");
    if (j->total_tokens > kMaxTokens) return fail(UH_ERR_UNSUPPORTED, "total_tokens exceeds 2^31-1");
    if (j->max_len != mx) return fail(UH_ERR_DIM, "max_len does not match the offsets");
    if (need_device && j->num_seqs > 0 && !j->offsets) return fail(UH_ERR_NULL, "device offsets NULL");
    return UH_OK;
}

uh_status check_mask(uh_mask m) {
    if (m.window < 0 || m.n_global < 0) return fail(UH_ERR_DOMAIN, "window and n_global must be >= 0");
    return UH_OK;
}

uh_status check_desc(const uh_attn_desc* d, uh_dtype dt) {
    if (!d) return fail(UH_ERR_NULL, "attention descriptor is NULL");
    if (dt != UH_BF16 && dt != UH_F32) return fail(UH_ERR_DOMAIN, "unknown dtype");
    if (d->num_heads < 1) return fail(UH_ERR_DOMAIN, "num_heads < 1");
    if (d->head_dim != 32 && d->head_dim != 64 && d->head_dim != 128)
        return fail(UH_ERR_SHAPE, "head_dim must be 32, 64 or 128");
    if (dt == UH_BF16 && d->head_dim != 128) return fail(UH_ERR_UNSUPPORTED, "bf16 path requires head_dim == 128");
    if (!(d->norm_n > 0.f)) return fail(UH_ERR_DOMAIN, "norm_n must be > 0");
    if (d->pos_bias && d->pos_bias_len < 1) return fail(UH_ERR_DOMAIN, "pos_bias_len < 1");
    if (d->time_bias) {
        if (d->time_bias_len < 1 || d->time_bias_len > 32) return fail(UH_ERR_DOMAIN, "time_bias_len must be in [1,32]");
        if (!d->timestamps) return fail(UH_ERR_NULL, "timestamps required with time_bias");
    }
    return UH_OK;
}

uh_status check_ptr(const void* p, const char* what, bool required = true) {
    if (!p) return required ? fail(UH_ERR_NULL, std::string(what) + " is NULL") : UH_OK;
    if (!aligned16(p)) return fail(UH_ERR_ALIGNMENT, std::string(what) + " not 16-byte aligned");
    return UH_OK;
}

uh_status check_ld(int64_t ld, int64_t width, uh_dtype dt, const char* what) {
    if (ld < width) return fail(UH_ERR_DIM, std::string(what) + ": row stride smaller than the row width");
    if (ld % ld_mult(dt)) return fail(UH_ERR_ALIGNMENT, std::string(what) + ": row stride not a multiple of 16 bytes");
    return UH_OK;
}

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------- layer workspace
struct LayerWs {
    size_t xh, uvqk, g, dy, ybuf, da, dh, dxh, attn_buf, stats, attn_ws, total;
};

LayerWs layer_ws(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dt, int backward) {
    LayerWs w{};
    const int64_t T = jag->total_tokens;
    const int d = p->attn.num_heads * p->attn.head_dim;
    const size_t es = esize(dt);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += a256(bytes); return o; };
    w.xh = take(T * d * es);
    w.uvqk = take(T * 4 * d * es);
    if (!backward) {
        w.ybuf = take(T * d * es);
        w.attn_buf = take(T * d * es);
        w.stats = take(4 * T * sizeof(float));
    } else {
        w.g = take(T * 4 * d * es);
        w.dy = take(T * d * es);
        w.ybuf = take(T * d * es);
        w.da = take(T * d * es);
        w.dh = take(T * 4 * d * es);
        w.dxh = take(T * d * es);
    }
    w.attn_ws = take(attn_ws_bytes(jag, m, &p->attn, dt, backward));
    w.total = off;
    return w;
}

uh_status check_layer(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dt,
                      bool need_device = true) {
    UH_TRY(check_jagged(jag, need_device));
    UH_TRY(check_mask(m));
    if (!p) return fail(UH_ERR_NULL, "layer params NULL");
    UH_TRY(check_desc(&p->attn, dt));
    const int d = p->attn.num_heads * p->attn.head_dim;
    if (dt == UH_BF16 && d % 64) return fail(UH_ERR_SHAPE, "bf16 layer requires d % 64 == 0");
    // the row kernels (norm.cu) hold a row in registers: 8 x 16-byte vectors per lane at most
    if (d > (dt == UH_BF16 ? 2048 : 1024)) return fail(UH_ERR_UNSUPPORTED, "layer d above the norm kernels' limit");
    UH_TRY(check_ptr(p->ln1_w, "ln1_w")); UH_TRY(check_ptr(p->ln1_b, "ln1_b"));
    UH_TRY(check_ptr(p->ln2_w, "ln2_w")); UH_TRY(check_ptr(p->ln2_b, "ln2_b"));
    UH_TRY(check_ptr(p->w1, "w1")); UH_TRY(check_ptr(p->w2, "w2"));
    UH_TRY(check_ptr(p->b1, "b1", false)); UH_TRY(check_ptr(p->b2, "b2", false));
    if (!(p->eps > 0.f)) return fail(UH_ERR_DOMAIN, "eps must be > 0");
    return UH_OK;
}

// Fingerprint of what a saved set depends on (FNV-1a over the host offsets, the mask and
// the attention descriptor's shape and scalars): uh_layer_fwd writes it, uh_layer_bwd
// rejects a saved set whose fingerprint differs (UH_ERR_CACHE_MISMATCH).
uint64_t saved_fingerprint(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dt) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* data, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(data);
        for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ull; }
    };
    mix(&jag->num_seqs, sizeof(jag->num_seqs));
    mix(&jag->total_tokens, sizeof(jag->total_tokens));
    mix(jag->host_offsets, sizeof(int32_t) * (size_t)(jag->num_seqs + 1));
    mix(&m, sizeof(m));
    const uh_attn_desc& a = p->attn;
    const int32_t shape[6] = {a.num_heads, a.head_dim, a.pos_bias ? a.pos_bias_len : 0,
                              a.time_bias ? a.time_bias_len : 0, (int32_t)dt, 0};
    mix(shape, sizeof(shape));
    mix(&a.alpha, sizeof(float)); mix(&a.norm_n, sizeof(float)); mix(&p->eps, sizeof(float));
    return h | 1ull;   // never 0: a zeroed (never-written) saved set always mismatches
}

}  // namespace

uh_status uh::validate_jagged(const uh_jagged* j, bool need_device) { return check_jagged(j, need_device); }

// =====================================================================================
extern "C" {

const char* uh_status_string(uh_status s) {
    switch (s) {
        case UH_OK: return "UH_OK";
        case UH_ERR_DIM: return "UH_ERR_DIM";
        case UH_ERR_DOMAIN: return "UH_ERR_DOMAIN";
        case UH_ERR_SHAPE: return "UH_ERR_SHAPE";
        case UH_ERR_CACHE_MISMATCH: return "UH_ERR_CACHE_MISMATCH";
        case UH_ERR_ALIGNMENT: return "UH_ERR_ALIGNMENT";
        case UH_ERR_WORKSPACE: return "UH_ERR_WORKSPACE";
        case UH_ERR_UNSUPPORTED: return "UH_ERR_UNSUPPORTED";
        case UH_ERR_CUDA: return "UH_ERR_CUDA";
        case UH_ERR_NULL: return "UH_ERR_NULL";
    }
    return "UH_ERR_UNKNOWN";
}

const char* uh_last_error(void);  // defined below (needs the thread-local in runtime.cu)

int uh_abi_version(void) { return UH_ABI_VERSION; }

int64_t uh_mask_nnz(uh_mask m, int64_t L) {
    if (L <= 0) return 0;
    const int64_t K1 = m.window, K2 = m.n_global;
    if (K1 >= L - 1) return L * (L + 1) / 2;
    // band: query q sees min(q, K1) + 1 keys; global prefix adds min(K2, q - K1) for q > K1
    const int64_t mm = std::min(L, K1 + 1);
    int64_t n = mm * (mm + 1) / 2 + (L - mm) * (K1 + 1);
    const int64_t R = L - 1 - K1;
    if (R > 0) {
        const int64_t m2 = std::min(R, K2);
        n += m2 * (m2 + 1) / 2 + (R - m2) * K2;
    }
    return n;
}

int64_t uh_batch_nnz(const uh_jagged* jag, uh_mask m) {
    if (!jag || !jag->host_offsets) return 0;
    int64_t n = 0;
    for (int b = 0; b < jag->num_seqs; ++b) n += uh_mask_nnz(m, jag->host_offsets[b + 1] - jag->host_offsets[b]);
    return n;
}

uh_status uh_attn_workspace_bytes(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dtype,
                                  int backward, size_t* bytes) {
    UH_TRY(check_jagged(jag, false));
    UH_TRY(check_mask(m));
    UH_TRY(check_desc(desc, dtype));
    if (!bytes) return fail(UH_ERR_NULL, "bytes is NULL");
    *bytes = attn_ws_bytes(jag, m, desc, dtype, backward);
    return UH_OK;
}

static uh_status check_attn_io(const uh_jagged* jag, const uh_attn_desc* desc, uh_dtype dt, const void* q,
                               const void* k, const void* v, int64_t ld_qkv) {
    const int64_t width = (int64_t)desc->num_heads * desc->head_dim;
    UH_TRY(check_ptr(q, "q")); UH_TRY(check_ptr(k, "k")); UH_TRY(check_ptr(v, "v"));
    UH_TRY(check_ld(ld_qkv, width, dt, "ld_qkv"));
    UH_TRY(check_ptr(desc->pos_bias, "pos_bias", false));
    UH_TRY(check_ptr(desc->time_bias, "time_bias", false));
    (void)jag;
    return UH_OK;
}

uh_status uh_attn_fwd(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dtype, const void* q,
                      const void* k, const void* v, int64_t ld_qkv, void* out, int64_t ld_out, void* ws,
                      size_t ws_bytes, void* stream) {
    UH_TRY(check_jagged(jag));
    UH_TRY(check_mask(m));
    UH_TRY(check_desc(desc, dtype));
    if (jag->total_tokens == 0) return UH_OK;
    UH_TRY(check_attn_io(jag, desc, dtype, q, k, v, ld_qkv));
    UH_TRY(check_ptr(out, "out"));
    UH_TRY(check_ld(ld_out, (int64_t)desc->num_heads * desc->head_dim, dtype, "ld_out"));
    const size_t need = attn_ws_bytes(jag, m, desc, dtype, 0);
    if (!ws || ws_bytes < need) return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    AttnCall c{};
    c.jag = jag; c.mask = m; c.desc = desc;
    c.q = q; c.k = k; c.v = v; c.ld_qkv = ld_qkv;
    c.out = out; c.ld_out = ld_out;
    c.ws = ws; c.ws_bytes = ws_bytes; c.st = (cudaStream_t)stream;
    return attn_fwd_run(c, dtype);
}

uh_status uh_attn_bwd(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dtype, const void* q,
                      const void* k, const void* v, int64_t ld_qkv, const void* dout, int64_t ld_dout, void* dq,
                      void* dk, void* dv, int64_t ld_grad, float* dpos_bias, float* dtime_bias, void* ws,
                      size_t ws_bytes, void* stream) {
    UH_TRY(check_jagged(jag));
    UH_TRY(check_mask(m));
    UH_TRY(check_desc(desc, dtype));
    if (jag->total_tokens == 0) return UH_OK;
    const int64_t width = (int64_t)desc->num_heads * desc->head_dim;
    UH_TRY(check_attn_io(jag, desc, dtype, q, k, v, ld_qkv));
    UH_TRY(check_ptr(dout, "dout"));
    UH_TRY(check_ptr(dq, "dq")); UH_TRY(check_ptr(dk, "dk")); UH_TRY(check_ptr(dv, "dv"));
    UH_TRY(check_ld(ld_dout, width, dtype, "ld_dout"));
    UH_TRY(check_ld(ld_grad, width, dtype, "ld_grad"));
    const size_t need = attn_ws_bytes(jag, m, desc, dtype, 1);
    if (!ws || ws_bytes < need) return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    AttnCall c{};
    c.jag = jag; c.mask = m; c.desc = desc;
    c.q = q; c.k = k; c.v = v; c.ld_qkv = ld_qkv;
    c.dout = dout; c.ld_dout = ld_dout;
    c.dq = dq; c.dk = dk; c.dv = dv; c.ld_grad = ld_grad;
    c.dpos = desc->pos_bias ? dpos_bias : nullptr;
    c.dts = desc->time_bias ? dtime_bias : nullptr;
    c.ws = ws; c.ws_bytes = ws_bytes; c.st = (cudaStream_t)stream;
    return attn_bwd_run(c, dtype);
}

// ------------------------------------------------------------------ layer
uh_status uh_layer_workspace_bytes(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dtype,
                                   int backward, size_t* bytes) {
    UH_TRY(check_layer(jag, m, p, dtype, false));
    if (!bytes) return fail(UH_ERR_NULL, "bytes is NULL");
    *bytes = layer_ws(jag, m, p, dtype, backward).total;
    return UH_OK;
}

uh_status uh_layer_fwd(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dtype, const void* x,
                       void* out, uh_layer_saved* saved, void* ws, size_t ws_bytes, void* stream) {
    UH_TRY(check_layer(jag, m, p, dtype));
    const int64_t T = jag->total_tokens;
    if (T == 0) return UH_OK;
    UH_TRY(check_ptr(x, "x")); UH_TRY(check_ptr(out, "out"));
    if (saved) {
        UH_TRY(check_ptr(saved->attn, "saved.attn"));
        if (!saved->ln1_mean || !saved->ln1_rstd || !saved->ln2_mean || !saved->ln2_rstd)
            return fail(UH_ERR_NULL, "saved statistics NULL");
    }
    const LayerWs w = layer_ws(jag, m, p, dtype, 0);
    if (!ws || ws_bytes < w.total) return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(w.total));
    cudaStream_t st = (cudaStream_t)stream;
    const int d = p->attn.num_heads * p->attn.head_dim;
    const size_t es = esize(dtype);
    uint8_t* W = (uint8_t*)ws;
    void* xh = W + w.xh;
    uint8_t* uvqk = W + w.uvqk;
    void* ybuf = W + w.ybuf;
    void* A = saved ? saved->attn : (void*)(W + w.attn_buf);
    float* st4 = (float*)(W + w.stats);
    float* mu1 = saved ? saved->ln1_mean : st4;
    float* rs1 = saved ? saved->ln1_rstd : st4 + T;
    float* mu2 = saved ? saved->ln2_mean : st4 + 2 * T;
    float* rs2 = saved ? saved->ln2_rstd : st4 + 3 * T;

    // F1: x^ = LN(x)                                                      (Eq. 1)
    UH_TRY(ln_fwd(dtype, T, d, x, d, p->ln1_w, p->ln1_b, p->eps, xh, d, mu1, rs1, st));
    // F2: UVQK = silu(x^ W1 + b1)                                         (Eq. 2)
    GemmDesc g1;
    g1.M = (int)T; g1.N = 4 * d; g1.K = d;
    g1.A = xh; g1.lda = d; g1.a_mn = false;
    g1.B = p->w1; g1.ldb = 4 * d; g1.b_mn = true;
    g1.epi = EPI_SILU; g1.out0 = uvqk; g1.ld0 = 4 * d; g1.bias = p->b1;
    UH_TRY(gemm_run(g1, dtype, st));
    // F3-F5: A = attention(Q, K, V)                                       (Eq. 3)
    AttnCall c{};
    c.jag = jag; c.mask = m; c.desc = &p->attn;
    c.q = uvqk + 2 * d * es; c.k = uvqk + 3 * d * es; c.v = uvqk + 1 * d * es; c.ld_qkv = 4 * d;
    c.out = A; c.ld_out = d;
    c.ws = W + w.attn_ws; c.ws_bytes = w.total - w.attn_ws; c.st = st;
    UH_TRY(attn_fwd_run(c, dtype));
    // F6: Y = LN(A) (.) U                                                 (Eq. 4, inner)
    UH_TRY(gated_norm_fwd(dtype, T, d, A, d, uvqk, 4 * d, p->ln2_w, p->ln2_b, p->eps, ybuf, d, mu2, rs2, st));
    // F7: out = Y W2 + b2 + x                                             (Eqs. 4-5)
    GemmDesc g2;
    g2.M = (int)T; g2.N = d; g2.K = d;
    g2.A = ybuf; g2.lda = d; g2.a_mn = false;
    g2.B = p->w2; g2.ldb = d; g2.b_mn = true;
    g2.epi = EPI_BF16; g2.out0 = out; g2.ld0 = d; g2.bias = p->b2; g2.resid = x; g2.ldr = d;
    UH_TRY(gemm_run(g2, dtype, st));
    if (saved) saved->fingerprint = saved_fingerprint(jag, m, p, dtype);
    return UH_OK;
}

uh_status uh_layer_bwd(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dtype, const void* x,
                       const uh_layer_saved* saved, const void* dout, void* dx, uh_layer_grads* grads, int accumulate,
                       void* ws, size_t ws_bytes, void* stream) {
    UH_TRY(check_layer(jag, m, p, dtype));
    if (!saved) return fail(UH_ERR_CACHE_MISMATCH, "backward needs the saved set of uh_layer_fwd");
    if (!saved->attn || !saved->ln1_mean || !saved->ln1_rstd || !saved->ln2_mean || !saved->ln2_rstd)
        return fail(UH_ERR_CACHE_MISMATCH, "saved set incomplete");
    if (saved->fingerprint != saved_fingerprint(jag, m, p, dtype))
        return fail(UH_ERR_CACHE_MISMATCH, "saved set was written by a forward with a different batch, mask or "
                                           "attention descriptor");
    if (!grads) return fail(UH_ERR_NULL, "grads NULL");
    if (!grads->ln1_w || !grads->ln1_b || !grads->w1 || !grads->ln2_w || !grads->ln2_b || !grads->w2)
        return fail(UH_ERR_NULL, "required parameter gradient NULL");
    if ((p->b1 && !grads->b1) || (p->b2 && !grads->b2))
        return fail(UH_ERR_NULL, "bias gradient NULL for a present bias");
    UH_TRY(check_ptr(x, "x")); UH_TRY(check_ptr(dout, "dout")); UH_TRY(check_ptr(dx, "dx"));
    UH_TRY(check_ptr(saved->attn, "saved.attn"));
    const LayerWs w = layer_ws(jag, m, p, dtype, 1);
    if (!ws || ws_bytes < w.total) return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(w.total));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t T = jag->total_tokens;
    const int d = p->attn.num_heads * p->attn.head_dim;
    const size_t es = esize(dtype);
    if (!accumulate) {
        auto z = [&](float* ptr, size_t n) -> uh_status {
            if (ptr) UH_CUDA(cudaMemsetAsync(ptr, 0, n * sizeof(float), st));
            return UH_OK;
        };
        UH_TRY(z(grads->ln1_w, d)); UH_TRY(z(grads->ln1_b, d));
        UH_TRY(z(grads->w1, (size_t)d * 4 * d)); UH_TRY(z(p->b1 ? grads->b1 : nullptr, 4 * d));
        UH_TRY(z(grads->ln2_w, d)); UH_TRY(z(grads->ln2_b, d));
        UH_TRY(z(grads->w2, (size_t)d * d)); UH_TRY(z(p->b2 ? grads->b2 : nullptr, d));
        if (p->attn.pos_bias) UH_TRY(z(grads->pos_bias, p->attn.pos_bias_len));
        if (p->attn.time_bias) UH_TRY(z(grads->time_bias, p->attn.time_bias_len));
    }
    if (T == 0) return UH_OK;
    uint8_t* W = (uint8_t*)ws;
    void* xh = W + w.xh;
    uint8_t* uvqk = W + w.uvqk;
    uint8_t* G = W + w.g;
    void* dY = W + w.dy;
    void* ybuf = W + w.ybuf;
    void* dA = W + w.da;
    uint8_t* dH = W + w.dh;
    void* dxh = W + w.dxh;

    // B3 (remat): x^ from saved statistics, then UVQK and silu'(h) by rerunning f1
    UH_TRY(ln_apply(dtype, T, d, x, d, p->ln1_w, p->ln1_b, saved->ln1_mean, saved->ln1_rstd, xh, d, st));
    GemmDesc g1;
    g1.M = (int)T; g1.N = 4 * d; g1.K = d;
    g1.A = xh; g1.lda = d; g1.B = p->w1; g1.ldb = 4 * d; g1.b_mn = true;
    g1.epi = EPI_SILU; g1.out0 = uvqk; g1.ld0 = 4 * d; g1.out1 = G; g1.ld1 = 4 * d; g1.bias = p->b1;
    UH_TRY(gemm_run(g1, dtype, st));
    // B1: dY = dOut W2^T
    GemmDesc gy;
    gy.M = (int)T; gy.N = d; gy.K = d;
    gy.A = dout; gy.lda = d; gy.B = p->w2; gy.ldb = d; gy.b_mn = false;
    gy.epi = EPI_BF16; gy.out0 = dY; gy.ld0 = d;
    UH_TRY(gemm_run(gy, dtype, st));
    // B2: gated-norm backward; Y recomputed inside; dU (.) silu'(h_U) -> dH[:, 0:d] (no concat)
    UH_TRY(gated_norm_bwd(dtype, T, d, dY, d, saved->attn, d, uvqk, 4 * d, G, 4 * d, p->ln2_w, p->ln2_b,
                          saved->ln2_mean, saved->ln2_rstd, dA, d, dH, 4 * d, ybuf, d, grads->ln2_w, grads->ln2_b, st));
    // B1: dW2 = Y^T dOut ; db2 = sum dOut
    GemmDesc gw2;
    gw2.M = d; gw2.N = d; gw2.K = (int)T;
    gw2.A = ybuf; gw2.lda = d; gw2.a_mn = true; gw2.B = dout; gw2.ldb = d; gw2.b_mn = true;
    gw2.epi = EPI_F32; gw2.out0 = grads->w2; gw2.ld0 = d;
    const bool fuse_cs = dtype == UH_BF16 && d % 256 == 0;   // db2 / db1 from the dW GEMMs' staged B tiles
    if (p->b2 && fuse_cs) gw2.colsum = grads->b2;
    UH_TRY(gemm_run(gw2, dtype, st));
    if (p->b2 && !fuse_cs) UH_TRY(colsum(dtype, T, d, dout, d, grads->b2, st));
    // B4: attention backward -> dH[:, V|Q|K] (x silu'(h)), d rab
    AttnCall c{};
    c.jag = jag; c.mask = m; c.desc = &p->attn;
    c.q = uvqk + 2 * d * es; c.k = uvqk + 3 * d * es; c.v = uvqk + 1 * d * es; c.ld_qkv = 4 * d;
    c.dout = dA; c.ld_dout = d;
    c.dq = dH + 2 * d * es; c.dk = dH + 3 * d * es; c.dv = dH + 1 * d * es; c.ld_grad = 4 * d;
    c.gq = G + 2 * d * es; c.gk = G + 3 * d * es; c.gv = G + 1 * d * es; c.ld_gate = 4 * d;
    c.dpos = p->attn.pos_bias ? grads->pos_bias : nullptr;
    c.dts = p->attn.time_bias ? grads->time_bias : nullptr;
    c.ws = W + w.attn_ws; c.ws_bytes = w.total - w.attn_ws; c.st = st;
    UH_TRY(attn_bwd_run(c, dtype));
    // B5: dW1 = x^T dH ; db1 = sum dH ; dx^ = dH W1^T
    GemmDesc gw1;
    gw1.M = d; gw1.N = 4 * d; gw1.K = (int)T;
    gw1.A = xh; gw1.lda = d; gw1.a_mn = true; gw1.B = dH; gw1.ldb = 4 * d; gw1.b_mn = true;
    gw1.epi = EPI_F32; gw1.out0 = grads->w1; gw1.ld0 = 4 * d;
    if (p->b1 && fuse_cs) gw1.colsum = grads->b1;
    UH_TRY(gemm_run(gw1, dtype, st));
    if (p->b1 && !fuse_cs) UH_TRY(colsum(dtype, T, 4 * d, dH, 4 * d, grads->b1, st));
    GemmDesc gx;
    gx.M = (int)T; gx.N = d; gx.K = 4 * d;
    gx.A = dH; gx.lda = 4 * d; gx.B = p->w1; gx.ldb = 4 * d; gx.b_mn = false;
    gx.epi = EPI_BF16; gx.out0 = dxh; gx.ld0 = d;
    UH_TRY(gemm_run(gx, dtype, st));
    // B6: dx = LN_bwd(dx^) + dOut
    UH_TRY(ln_bwd(dtype, T, d, dxh, d, x, d, p->ln1_w, saved->ln1_mean, saved->ln1_rstd, dout, d, dx, d,
                  grads->ln1_w, grads->ln1_b, st));
    return UH_OK;
}

// ------------------------------------------------------------------ partitioner
uh_status uh_partition_lpt(const int32_t* lengths, int32_t B, int32_t world, uh_mask m, int32_t d, int32_t num_heads,
                           int32_t* rank_of_seq, double* rank_cost) {
    if (B < 0 || world < 1 || d < 1 || num_heads < 1) return fail(UH_ERR_DOMAIN, "bad partition arguments");
    UH_TRY(check_mask(m));
    if (B > 0 && (!lengths || !rank_of_seq)) return fail(UH_ERR_NULL, "lengths / rank_of_seq NULL");
    if (!rank_cost) return fail(UH_ERR_NULL, "rank_cost NULL");
    const int dh = d / num_heads;
    std::vector<double> cost(B);
    for (int i = 0; i < B; ++i) {
        if (lengths[i] < 0) return fail(UH_ERR_DOMAIN, "negative length");
        const double L = lengths[i];
        // the step's flops on this sequence: four f1-shaped GEMMs (f1, remat f1, dW1, dx^), three
        // f2-shaped (f2, dY, dW2), attention 4 d_h forward + 10 d_h backward per allowed pair-head
        cost[i] = 4.0 * (2.0 * L * d * 4 * d) + 3.0 * (2.0 * L * d * d) +
                  14.0 * dh * num_heads * (double)uh_mask_nnz(m, lengths[i]);
    }
    std::vector<int> order(B);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    std::vector<double> load(world, 0.0);
    for (int i : order) {
        int best = 0;
        for (int r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        rank_of_seq[i] = best;
        load[best] += cost[i];
    }
    for (int r = 0; r < world; ++r) rank_cost[r] = load[r];
    return UH_OK;
}

}  // extern "C"

#include "../../include/uhstu_testing.h"
extern "C" uh_status uh_test_gemm(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
                                  int64_t ldb, int b_mn, int epi, void* out0, int64_t ld0, void* out1, int64_t ld1,
                                  const float* bias, const void* resid, int64_t ldr, uh_dtype dtype, int cta_pair,
                                  void* stream) {
    if (M < 0 || N < 0 || K < 0 || epi < 0 || epi > 2 || cta_pair < 0 || cta_pair > 2)
        return fail(UH_ERR_DOMAIN, "bad gemm arguments");
    GemmDesc g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_mn = a_mn != 0;
    g.B = B; g.ldb = ldb; g.b_mn = b_mn != 0;
    g.epi = epi; g.out0 = out0; g.ld0 = ld0; g.out1 = out1; g.ld1 = ld1; g.bias = bias; g.resid = resid; g.ldr = ldr;
    g.pair = cta_pair;
    return gemm_run(g, dtype, (cudaStream_t)stream);
}

// ================================================================== NEXT-2: FP8 projections (uhstu_fp8.h)
#include "../../include/uhstu_fp8.h"

namespace {
uh_status check_codes_ld(int64_t ld, int64_t width, const char* what) {
    if (ld < width) return uh::fail(UH_ERR_DIM, std::string(what) + ": row stride smaller than the row width");
    if (ld % 16) return uh::fail(UH_ERR_ALIGNMENT, std::string(what) + ": code row stride not a multiple of 16 bytes");
    return UH_OK;
}
uh_status check_f32(const void* p, const char* what) {
    if (!p) return uh::fail(UH_ERR_NULL, std::string(what) + " is NULL");
    if (reinterpret_cast<uintptr_t>(p) % 4) return uh::fail(UH_ERR_ALIGNMENT, std::string(what) + " not 4-byte aligned");
    return UH_OK;
}
}  // namespace

extern "C" uh_status uh_ln_fwd_fp8(int64_t T, int d, const void* x, int64_t ldx, const float* w, const float* b,
                                   float eps, uint8_t* q, int64_t ldq, float* scale, float* mean, float* rstd,
                                   void* stream) {
    using namespace uh;
    if (T < 0 || d <= 0 || d % 8 || d > 2048) return fail(UH_ERR_DIM, "ln_fwd_fp8: T >= 0, 0 < d <= 2048, d % 8 == 0");
    if (T == 0) return UH_OK;
    UH_TRY(check_ptr(x, "x")); UH_TRY(check_ptr(w, "w")); UH_TRY(check_ptr(b, "b")); UH_TRY(check_ptr(q, "q"));
    UH_TRY(check_f32(scale, "scale"));
    UH_TRY(check_ld(ldx, d, UH_BF16, "ldx")); UH_TRY(check_codes_ld(ldq, d, "ldq"));
    return ln_fwd_fp8(T, d, x, ldx, w, b, eps, q, ldq, scale, mean, rstd, (cudaStream_t)stream);
}

extern "C" uh_status uh_gated_norm_fwd_fp8(int64_t T, int d, const void* A, int64_t lda, const void* U, int64_t ldu,
                                           const float* w, const float* b, float eps, uint8_t* q, int64_t ldq,
                                           float* scale, float* mean, float* rstd, void* stream) {
    using namespace uh;
    if (T < 0 || d <= 0 || d % 8 || d > 2048) return fail(UH_ERR_DIM, "gated_norm_fwd_fp8: T >= 0, 0 < d <= 2048, d % 8 == 0");
    if (T == 0) return UH_OK;
    UH_TRY(check_ptr(A, "A")); UH_TRY(check_ptr(U, "U")); UH_TRY(check_ptr(w, "w")); UH_TRY(check_ptr(b, "b"));
    UH_TRY(check_ptr(q, "q")); UH_TRY(check_f32(scale, "scale"));
    UH_TRY(check_ld(lda, d, UH_BF16, "lda")); UH_TRY(check_ld(ldu, d, UH_BF16, "ldu"));
    UH_TRY(check_codes_ld(ldq, d, "ldq"));
    return gated_norm_fwd_fp8(T, d, A, lda, U, ldu, w, b, eps, q, ldq, scale, mean, rstd, (cudaStream_t)stream);
}

extern "C" uh_status uh_quant_weight_fp8(int K, int N, const void* W, int64_t ldw, uint8_t* qt, int64_t ldq,
                                         float* scale, void* stream) {
    using namespace uh;
    if (K < 0 || N < 0) return fail(UH_ERR_DIM, "quant_weight_fp8: K, N >= 0");
    if (K == 0 || N == 0) return UH_OK;
    UH_TRY(check_ptr(W, "W")); UH_TRY(check_ptr(qt, "qt")); UH_TRY(check_f32(scale, "scale"));
    UH_TRY(check_ld(ldw, N, UH_BF16, "ldw")); UH_TRY(check_codes_ld(ldq, K, "ldq"));
    return quant_weight_fp8(K, N, W, ldw, qt, ldq, scale, (cudaStream_t)stream);
}

extern "C" uh_status uh_gemm_fp8(int M, int N, int K, const uint8_t* qa, int64_t lda, const float* sa,
                                 const uint8_t* qb, int64_t ldb, const float* sb, int epi, void* out, int64_t ldo,
                                 const float* bias, const void* resid, int64_t ldr, void* stream) {
    using namespace uh;
    if (M < 0 || N < 0 || K < 0) return fail(UH_ERR_DIM, "gemm_fp8: M, N, K >= 0");
    if (epi != 0 && epi != 1) return fail(UH_ERR_DOMAIN, "gemm_fp8: epi must be 0 (bf16 + bias + resid) or 1 (silu)");
    if (epi == 1 && resid) return fail(UH_ERR_DOMAIN, "gemm_fp8: the SiLU epilogue takes no residual");
    if (M == 0 || N == 0) return UH_OK;
    UH_TRY(check_ptr(qa, "qa")); UH_TRY(check_ptr(qb, "qb")); UH_TRY(check_ptr(out, "out"));
    UH_TRY(check_f32(sa, "sa")); UH_TRY(check_f32(sb, "sb"));
    UH_TRY(check_codes_ld(lda, K, "lda")); UH_TRY(check_codes_ld(ldb, K, "ldb"));
    UH_TRY(check_ld(ldo, N, UH_BF16, "ldo"));
    if (resid) { UH_TRY(check_ptr(resid, "resid")); UH_TRY(check_ld(ldr, N, UH_BF16, "ldr")); }
    GemmDesc g;
    g.M = M; g.N = N; g.K = K;
    g.A = qa; g.lda = lda; g.B = qb; g.ldb = ldb;
    g.epi = epi == 1 ? EPI_SILU : EPI_BF16;
    g.out0 = out; g.ld0 = ldo; g.bias = bias; g.resid = resid; g.ldr = ldr;
    return gemm_fp8_run(g, sa, sb, (cudaStream_t)stream);
}

extern "C" uh_status uh_layer_fwd_fp8(const uh_jagged* jag, uh_mask m, const uh_layer_params* p,
                                      const uh_fp8_weights* qw, const void* x, void* out, uh_layer_saved* saved,
                                      void* ws, size_t ws_bytes, void* stream) {
    using namespace uh;
    const uh_dtype dtype = UH_BF16;
    UH_TRY(check_layer(jag, m, p, dtype));
    if (!qw || !qw->w1t || !qw->s1 || !qw->w2t || !qw->s2) return fail(UH_ERR_NULL, "fp8 weights NULL");
    const int64_t T = jag->total_tokens;
    if (T == 0) return UH_OK;
    UH_TRY(check_ptr(x, "x")); UH_TRY(check_ptr(out, "out"));
    if (saved) {
        UH_TRY(check_ptr(saved->attn, "saved.attn"));
        if (!saved->ln1_mean || !saved->ln1_rstd || !saved->ln2_mean || !saved->ln2_rstd)
            return fail(UH_ERR_NULL, "saved statistics NULL");
    }
    const int d = p->attn.num_heads * p->attn.head_dim;
    if (d % 128) return fail(UH_ERR_UNSUPPORTED, "fp8 layer needs d % 128 == 0");
    const LayerWs w = layer_ws(jag, m, p, dtype, 0);
    if (!ws || ws_bytes < w.total) return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(w.total));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t es = 2;
    uint8_t* W = (uint8_t*)ws;
    uint8_t* codes = W + w.xh;            // [T][d] E4M3 (x^, then Y): fits the bf16 x^ slot
    float* rscale = (float*)(W + w.ybuf); // [T] row scales: fits the bf16 Y slot
    uint8_t* uvqk = W + w.uvqk;
    void* A = saved ? saved->attn : (void*)(W + w.attn_buf);
    float* st4 = (float*)(W + w.stats);
    float* mu1 = saved ? saved->ln1_mean : st4;
    float* rs1 = saved ? saved->ln1_rstd : st4 + T;
    float* mu2 = saved ? saved->ln2_mean : st4 + 2 * T;
    float* rs2 = saved ? saved->ln2_rstd : st4 + 3 * T;

    // F1 + quant: codes(x^), s_x                                           (Eq. 1)
    UH_TRY(ln_fwd_fp8(T, d, x, d, p->ln1_w, p->ln1_b, p->eps, codes, d, rscale, mu1, rs1, st));
    // F2: UVQK = silu(s_x (q_x q_W1^T) s_W1 + b1)                          (Eq. 2)
    GemmDesc g1;
    g1.M = (int)T; g1.N = 4 * d; g1.K = d;
    g1.A = codes; g1.lda = d; g1.B = qw->w1t; g1.ldb = d;
    g1.epi = EPI_SILU; g1.out0 = uvqk; g1.ld0 = 4 * d; g1.bias = p->b1;
    UH_TRY(gemm_fp8_run(g1, rscale, qw->s1, st));
    // F3-F5: A = attention(Q, K, V), bf16                                  (Eq. 3)
    AttnCall c{};
    c.jag = jag; c.mask = m; c.desc = &p->attn;
    c.q = uvqk + 2 * d * es; c.k = uvqk + 3 * d * es; c.v = uvqk + 1 * d * es; c.ld_qkv = 4 * d;
    c.out = A; c.ld_out = d;
    c.ws = W + w.attn_ws; c.ws_bytes = w.total - w.attn_ws; c.st = st;
    UH_TRY(attn_fwd_run(c, dtype));
    // F6 + quant: codes(Y), s_Y with Y = LN(A) (.) U                      (Eq. 4 inner)
    UH_TRY(gated_norm_fwd_fp8(T, d, A, d, uvqk, 4 * d, p->ln2_w, p->ln2_b, p->eps, codes, d, rscale, mu2, rs2, st));
    // F7: out = s_Y (q_Y q_W2^T) s_W2 + b2 + x                             (Eqs. 4-5)
    GemmDesc g2;
    g2.M = (int)T; g2.N = d; g2.K = d;
    g2.A = codes; g2.lda = d; g2.B = qw->w2t; g2.ldb = d;
    g2.epi = EPI_BF16; g2.out0 = out; g2.ld0 = d; g2.bias = p->b2; g2.resid = x; g2.ldr = d;
    UH_TRY(gemm_fp8_run(g2, rscale, qw->s2, st));
    if (saved) saved->fingerprint = saved_fingerprint(jag, m, p, dtype);
    return UH_OK;
}
