// C-ABI entry points for convolution and attention: validate, pick the
// algorithm, launch.
//
// Algorithm policy.  bf16 (and fp32, via the exact bf16x3 split) runs on the
// tcgen05 kernels whenever the geometry is inside their envelope.  The
// CUDA-core kernels exist for what the tensor cores cannot do exactly — fp64
// (the reference's default dtype) — and for geometries outside the envelope
// (strides > 1, 1-D convs, channel counts that are not multiples of 16, ...),
// which the reference's own test-suite exercises.  They are never a silent
// detour for the hot path: every call routed to them is counted
// (dp_simt_count), DP_ALGO_STRICT refuses them for bf16/fp32, and the
// sharded-conv parity tests and bench.py assert the count stays 0.
#include "common.cuh"

namespace dp {
int conv_fwd_simt_launch(const dp_conv_geom *, int, const void *, const void *, const void *,
                         void *, cudaStream_t);
int conv_dgrad_simt_launch(const dp_conv_geom *, int, const void *, const void *, void *, void *,
                           cudaStream_t);
int64_t conv_wgrad_simt_workspace(const dp_conv_geom *, int);
int conv_wgrad_simt_launch(const dp_conv_geom *, int, const void *, const void *, const void *,
                           void *, void *, int64_t, cudaStream_t);
int attn_fwd_update_simt_launch(const dp_attn_geom *, int, const void *, const void *,
                                const void *, void *, void *, void *, cudaStream_t);
int attn_bwd_update_simt_launch(const dp_attn_geom *, int, const void *, const void *,
                                const void *, const void *, const void *, const void *, void *,
                                void *, void *, cudaStream_t);
// tcgen05 paths (conv_tc.cu / attn_tc.cu)
int conv_tc_eligible(const dp_conv_geom *, int dtype, int which);
int64_t conv_tc_workspace(const dp_conv_geom *, int which);
int conv_fwd_tc_launch(const dp_conv_geom *, const void *, const void *, const void *, void *,
                       void *, int64_t, cudaStream_t);
int conv_dgrad_tc_launch(const dp_conv_geom *, const void *, const void *, void *, void *,
                         void *, int64_t, cudaStream_t);
int conv_wgrad_tc_launch(const dp_conv_geom *, const void *, const void *, const void *, void *,
                         void *, int64_t, cudaStream_t);
int attn_tc_eligible(const dp_attn_geom *, int dtype);
int attn_bwd_tc_eligible(const dp_attn_geom *, int dtype);
int attn_fwd_update_tc_launch(const dp_attn_geom *, const void *, const void *, const void *,
                              void *, void *, void *, cudaStream_t);
int attn_bwd_update_tc_launch(const dp_attn_geom *, const void *, const void *, const void *,
                              const void *, const void *, const void *, void *, void *, void *,
                              cudaStream_t);
}  // namespace dp

namespace dp {
int conv_x3_eligible(const dp_conv_geom *, int which);
int64_t conv_x3_workspace(const dp_conv_geom *, int which);
int conv_x3_launch(const dp_conv_geom *, int which, const void *, const void *, const void *, void *,
                   void *, void *, int64_t, cudaStream_t);
int64_t conv_x3_parts_workspace(const dp_conv_geom *, int which);
int64_t conv_x3_operand_bytes(const dp_conv_geom *, int operand);
int conv_x3_split(const dp_conv_geom *, int operand, const void *, void *, cudaStream_t);
int conv_x3_parts_launch(const dp_conv_geom *, int which, const void *, const void *, const void *,
                         void *, void *, void *, int64_t, cudaStream_t);
}  // namespace dp

using namespace dp;

// fp32 convs go to the bf16x3 tensor-core path (conv_x3.cu) when it covers
// the shape (auto / tc), else to the CUDA-core kernels
static int eligible_tc(const dp_conv_geom *g, int dtype, int which) {
    if (dtype == DP_F32) return conv_x3_eligible(g, which);
    return conv_tc_eligible(g, dtype, which);
}

static unsigned long long g_simt_calls = 0;

static int pick(int algo, int eligible, const char *what, int dtype, bool count = true) {
    int a;
    if (algo == DP_ALGO_SIMT) {
        a = DP_ALGO_SIMT;
    } else if (algo == DP_ALGO_TC || (algo == DP_ALGO_STRICT && dtype != DP_F64)) {
        if (!eligible) {
            set_error("%s: configuration outside the tcgen05 envelope", what);
            return -1;
        }
        a = DP_ALGO_TC;
    } else {
        a = eligible ? DP_ALGO_TC : DP_ALGO_SIMT;
    }
    if (count && a == DP_ALGO_SIMT) __atomic_add_fetch(&g_simt_calls, 1ull, __ATOMIC_RELAXED);
    return a;
}

extern "C" uint64_t dp_simt_count(void) {
    return __atomic_load_n(&g_simt_calls, __ATOMIC_RELAXED);
}

extern "C" int64_t dp_conv_workspace(const dp_conv_geom *g, int dtype, int algo, int which) {
    int a = pick(algo, eligible_tc(g, dtype, which), "dp_conv_workspace", dtype, false);
    if (a < 0) return -1;
    if (a == DP_ALGO_TC)
        return dtype == DP_F32 ? conv_x3_workspace(g, which) : conv_tc_workspace(g, which);
    return which == DP_CONV_WGRAD ? conv_wgrad_simt_workspace(g, dtype) : 0;
}

extern "C" int dp_conv_fwd(const dp_conv_geom *g, int dtype, int algo, const void *x,
                           const void *xh, const void *w, void *y, void *ws, int64_t ws_bytes,
                           void *stream) {
    int a = pick(algo, eligible_tc(g, dtype, DP_CONV_FWD), "dp_conv_fwd", dtype);
    if (a < 0) return DP_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if (a == DP_ALGO_TC && dtype == DP_F32)
        return conv_x3_launch(g, DP_CONV_FWD, x, xh, w, y, nullptr, ws, ws_bytes, st);
    if (a == DP_ALGO_TC) return conv_fwd_tc_launch(g, x, xh, w, y, ws, ws_bytes, st);
    return conv_fwd_simt_launch(g, dtype, x, xh, w, y, st);
}

extern "C" int dp_conv_dgrad(const dp_conv_geom *g, int dtype, int algo, const void *dy,
                             const void *w, void *dx, void *dxh, void *ws, int64_t ws_bytes,
                             void *stream) {
    int a = pick(algo, eligible_tc(g, dtype, DP_CONV_DGRAD), "dp_conv_dgrad", dtype);
    if (a < 0) return DP_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if (a == DP_ALGO_TC && dtype == DP_F32)
        return conv_x3_launch(g, DP_CONV_DGRAD, dy, nullptr, w, dx, dxh, ws, ws_bytes, st);
    if (a == DP_ALGO_TC) return conv_dgrad_tc_launch(g, dy, w, dx, dxh, ws, ws_bytes, st);
    return conv_dgrad_simt_launch(g, dtype, dy, w, dx, dxh, st);
}

extern "C" int dp_conv_wgrad(const dp_conv_geom *g, int dtype, int algo, const void *x,
                             const void *xh, const void *dy, void *dw, void *ws, int64_t ws_bytes,
                             void *stream) {
    int a = pick(algo, eligible_tc(g, dtype, DP_CONV_WGRAD), "dp_conv_wgrad", dtype);
    if (a < 0) return DP_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if (a == DP_ALGO_TC && dtype == DP_F32)
        return conv_x3_launch(g, DP_CONV_WGRAD, x, xh, dy, dw, nullptr, ws, ws_bytes, st);
    if (a == DP_ALGO_TC) return conv_wgrad_tc_launch(g, x, xh, dy, dw, ws, ws_bytes, st);
    return conv_wgrad_simt_launch(g, dtype, x, xh, dy, dw, ws, ws_bytes, st);
}

// bf16x3 with caller-held split operands: tcgen05 only (no CUDA-core form)
extern "C" int64_t dp_conv_x3_operand_bytes(const dp_conv_geom *g, int operand) {
    return conv_x3_operand_bytes(g, operand);
}
extern "C" int dp_conv_x3_split(const dp_conv_geom *g, int operand, const void *src, void *parts,
                                void *stream) {
    return conv_x3_split(g, operand, src, parts, (cudaStream_t)stream);
}
extern "C" int64_t dp_conv_x3_parts_workspace(const dp_conv_geom *g, int which) {
    return conv_x3_parts_workspace(g, which);
}
extern "C" int dp_conv_x3_fwd_parts(const dp_conv_geom *g, const void *xp, const void *xhp,
                                    const void *w, void *y, void *ws, int64_t ws_bytes,
                                    void *stream) {
    return conv_x3_parts_launch(g, DP_CONV_FWD, xp, xhp, w, y, nullptr, ws, ws_bytes,
                                (cudaStream_t)stream);
}
extern "C" int dp_conv_x3_dgrad_parts(const dp_conv_geom *g, const void *dyp, const void *w,
                                      void *dx, void *dxh, void *ws, int64_t ws_bytes,
                                      void *stream) {
    return conv_x3_parts_launch(g, DP_CONV_DGRAD, dyp, nullptr, w, dx, dxh, ws, ws_bytes,
                                (cudaStream_t)stream);
}
extern "C" int dp_conv_x3_wgrad_parts(const dp_conv_geom *g, const void *xp, const void *xhp,
                                      const void *dyp, void *dw, void *ws, int64_t ws_bytes,
                                      void *stream) {
    return conv_x3_parts_launch(g, DP_CONV_WGRAD, xp, xhp, dyp, dw, nullptr, ws, ws_bytes,
                                (cudaStream_t)stream);
}

extern "C" int dp_attn_fwd_update(const dp_attn_geom *g, int dtype, int algo, const void *q,
                                  const void *k, const void *v, void *m, void *l, void *acc,
                                  void *stream) {
    int a = pick(algo, attn_tc_eligible(g, dtype), "dp_attn_fwd_update", dtype);
    if (a < 0) return DP_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if (a == DP_ALGO_TC) return attn_fwd_update_tc_launch(g, q, k, v, m, l, acc, st);
    return attn_fwd_update_simt_launch(g, dtype, q, k, v, m, l, acc, st);
}

extern "C" int dp_attn_bwd_update(const dp_attn_geom *g, int dtype, int algo, const void *q,
                                  const void *k, const void *v, const void *dout,
                                  const void *lse, const void *delta, void *dq, void *dk,
                                  void *dv, void *stream) {
    int a = pick(algo, attn_bwd_tc_eligible(g, dtype), "dp_attn_bwd_update", dtype);
    if (a < 0) return DP_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if (a == DP_ALGO_TC)
        return attn_bwd_update_tc_launch(g, q, k, v, dout, lse, delta, dq, dk, dv, st);
    return attn_bwd_update_simt_launch(g, dtype, q, k, v, dout, lse, delta, dq, dk, dv, st);
}
