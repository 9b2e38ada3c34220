// Ring-attention block kernels on CUDA cores (general dtype path).
//
// One warp owns one (row, head) pair; lanes split the head dim.  These are
// the fp32/fp64 parity path (the reference keeps its softmax state in fp64,
// domainpar/ops.py:199-214) and the fallback for shapes outside the
// tcgen05 attention kernel (attn_tc.cu).  The online-softmax fold is the
// reference's RingSoftmaxState.update restated per key block.
//
// State precision: fp64 for fp32/fp64 inputs (as the reference), fp32 for
// bf16 inputs.
#include "common.cuh"

namespace dp {
namespace {

template <typename T> struct StateT { using type = double; };
template <> struct StateT<__nv_bfloat16> { using type = float; };

constexpr int kMaxPerLane = 8;  // head dim <= 256

struct AG {
    int64_t sq, sk, H, D;
    int64_t q_rs, q_hs, k_rs, k_hs, v_rs, v_hs, o_rs, o_hs;
    double scale;
};

AG make_ag(const dp_attn_geom *g) {
    AG a;
    a.sq = g->sq; a.sk = g->sk; a.H = g->heads; a.D = g->dim;
    a.q_rs = g->q_rs; a.q_hs = g->q_hs; a.k_rs = g->k_rs; a.k_hs = g->k_hs;
    a.v_rs = g->v_rs; a.v_hs = g->v_hs; a.o_rs = g->o_rs; a.o_hs = g->o_hs;
    a.scale = g->scale;
    return a;
}

template <typename S>
__device__ __forceinline__ S warp_sum(S v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ void load_row(const T *p, int64_t D, int lane,
                                         typename StateT<T>::type (&r)[kMaxPerLane]) {
#pragma unroll
    for (int j = 0; j < kMaxPerLane; ++j) {
        int64_t d = lane + 32 * j;
        r[j] = d < D ? (typename StateT<T>::type)to_acc(p[d]) : 0;
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
attn_fwd_update_simt(AG g, const T *__restrict__ q, const T *__restrict__ k,
                     const T *__restrict__ v, typename StateT<T>::type *__restrict__ m,
                     typename StateT<T>::type *__restrict__ l,
                     typename StateT<T>::type *__restrict__ acc) {
    using S = typename StateT<T>::type;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
         row < g.sq * g.H; row += nw) {
        const int64_t i = row / g.H, h = row % g.H;
        S qr[kMaxPerLane], ar[kMaxPerLane];
        load_row(q + i * g.q_rs + h * g.q_hs, g.D, lane, qr);
        S *ap = acc + row * g.D;
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) {
            int64_t d = lane + 32 * j;
            ar[j] = d < g.D ? ap[d] : 0;
        }
        S mr = m[row], lr = l[row];
        // pass 1: block row max (as the reference: m_new = max(m, rowmax(s)))
        S bmax = neg_inf<S>();
        for (int64_t kj = 0; kj < g.sk; ++kj) {
            S kr[kMaxPerLane];
            load_row(k + kj * g.k_rs + h * g.k_hs, g.D, lane, kr);
            S dot = 0;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) dot += qr[j] * kr[j];
            dot = warp_sum(dot) * (S)g.scale;
            bmax = dot > bmax ? dot : bmax;
        }
        const S mnew = mr > bmax ? mr : bmax;
        const S c = acc_exp(mr - mnew);  // exp(-inf) = 0 on the first block
        S psum = 0;
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) ar[j] *= c;
        for (int64_t kj = 0; kj < g.sk; ++kj) {
            S kr[kMaxPerLane], vr[kMaxPerLane];
            load_row(k + kj * g.k_rs + h * g.k_hs, g.D, lane, kr);
            load_row(v + kj * g.v_rs + h * g.v_hs, g.D, lane, vr);
            S dot = 0;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) dot += qr[j] * kr[j];
            dot = warp_sum(dot) * (S)g.scale;
            S p = acc_exp(dot - mnew);
            psum += p;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) ar[j] += p * vr[j];
        }
        if (lane == 0) {
            m[row] = mnew;
            l[row] = lr * c + psum;
        }
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) {
            int64_t d = lane + 32 * j;
            if (d < g.D) ap[d] = ar[j];
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
attn_finalize_k(AG g, const typename StateT<T>::type *__restrict__ m,
                const typename StateT<T>::type *__restrict__ l,
                const typename StateT<T>::type *__restrict__ acc, T *__restrict__ out,
                typename StateT<T>::type *__restrict__ lse) {
    using S = typename StateT<T>::type;
    const int64_t total = g.sq * g.H * g.D;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t row = idx / g.D, d = idx % g.D;
        int64_t i = row / g.H, h = row % g.H;
        S lv = l[row];
        out[i * g.o_rs + h * g.o_hs + d] = from_acc<T>(acc[idx] / lv);
        if (d == 0 && lse) lse[row] = m[row] + acc_log(lv);
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
attn_delta_k(AG g, const T *__restrict__ o, const T *__restrict__ dout,
             typename StateT<T>::type *__restrict__ delta) {
    using S = typename StateT<T>::type;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
         row < g.sq * g.H; row += nw) {
        const int64_t i = row / g.H, h = row % g.H;
        S a[kMaxPerLane], b[kMaxPerLane];
        load_row(o + i * g.o_rs + h * g.o_hs, g.D, lane, a);
        load_row(dout + i * g.o_rs + h * g.o_hs, g.D, lane, b);
        S s = 0;
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) s += a[j] * b[j];
        s = warp_sum(s);
        if (lane == 0) delta[row] = s;
    }
}

// dQ for one K/V block: warp per (query row, head)
template <typename T>
__global__ void __launch_bounds__(256)
attn_bwd_dq_simt(AG g, const T *__restrict__ q, const T *__restrict__ k, const T *__restrict__ v,
                 const T *__restrict__ dout, const typename StateT<T>::type *__restrict__ lse,
                 const typename StateT<T>::type *__restrict__ delta,
                 typename StateT<T>::type *__restrict__ dq) {
    using S = typename StateT<T>::type;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
         row < g.sq * g.H; row += nw) {
        const int64_t i = row / g.H, h = row % g.H;
        S qr[kMaxPerLane], dor[kMaxPerLane], acc[kMaxPerLane];
        load_row(q + i * g.q_rs + h * g.q_hs, g.D, lane, qr);
        load_row(dout + i * g.o_rs + h * g.o_hs, g.D, lane, dor);
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) acc[j] = 0;
        const S L = lse[row], Dl = delta[row];
        for (int64_t kj = 0; kj < g.sk; ++kj) {
            S kr[kMaxPerLane], vr[kMaxPerLane];
            load_row(k + kj * g.k_rs + h * g.k_hs, g.D, lane, kr);
            load_row(v + kj * g.v_rs + h * g.v_hs, g.D, lane, vr);
            S s = 0, dp = 0;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) {
                s += qr[j] * kr[j];
                dp += dor[j] * vr[j];
            }
            s = warp_sum(s) * (S)g.scale;
            dp = warp_sum(dp);
            S p = acc_exp(s - L);
            S ds = p * (dp - Dl) * (S)g.scale;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) acc[j] += ds * kr[j];
        }
        S *out = dq + row * g.D;
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) {
            int64_t d = lane + 32 * j;
            if (d < g.D) out[d] += acc[j];
        }
    }
}

// dK, dV for one K/V block: warp per (key row, head)
template <typename T>
__global__ void __launch_bounds__(256)
attn_bwd_dkdv_simt(AG g, const T *__restrict__ q, const T *__restrict__ k,
                   const T *__restrict__ v, const T *__restrict__ dout,
                   const typename StateT<T>::type *__restrict__ lse,
                   const typename StateT<T>::type *__restrict__ delta,
                   typename StateT<T>::type *__restrict__ dk, typename StateT<T>::type *__restrict__ dv) {
    using S = typename StateT<T>::type;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
         row < g.sk * g.H; row += nw) {
        const int64_t kj = row / g.H, h = row % g.H;
        S kr[kMaxPerLane], vr[kMaxPerLane], ak[kMaxPerLane], av[kMaxPerLane];
        load_row(k + kj * g.k_rs + h * g.k_hs, g.D, lane, kr);
        load_row(v + kj * g.v_rs + h * g.v_hs, g.D, lane, vr);
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) ak[j] = av[j] = 0;
        for (int64_t i = 0; i < g.sq; ++i) {
            S qr[kMaxPerLane], dor[kMaxPerLane];
            load_row(q + i * g.q_rs + h * g.q_hs, g.D, lane, qr);
            load_row(dout + i * g.o_rs + h * g.o_hs, g.D, lane, dor);
            S s = 0, dp = 0;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) {
                s += qr[j] * kr[j];
                dp += dor[j] * vr[j];
            }
            s = warp_sum(s) * (S)g.scale;
            dp = warp_sum(dp);
            const int64_t qrow = i * g.H + h;
            S p = acc_exp(s - lse[qrow]);
            S ds = p * (dp - delta[qrow]) * (S)g.scale;
#pragma unroll
            for (int j = 0; j < kMaxPerLane; ++j) {
                av[j] += p * dor[j];
                ak[j] += ds * qr[j];
            }
        }
        S *pk = dk + row * g.D;
        S *pv = dv + row * g.D;
#pragma unroll
        for (int j = 0; j < kMaxPerLane; ++j) {
            int64_t d = lane + 32 * j;
            if (d < g.D) {
                pk[d] += ak[j];
                pv[d] += av[j];
            }
        }
    }
}

int check(const dp_attn_geom *g) {
    DP_REQUIRE(g, DP_ERR_INVALID, "attn: null geometry");
    DP_REQUIRE(g->dim >= 1 && g->dim <= 32 * kMaxPerLane, DP_ERR_UNSUPPORTED,
               "attn: head dim %lld outside [1, %d]", (long long)g->dim, 32 * kMaxPerLane);
    DP_REQUIRE(g->sq >= 0 && g->sk >= 0 && g->heads >= 1, DP_ERR_INVALID, "attn: sizes");
    return DP_OK;
}

}  // namespace

int attn_fwd_update_simt_launch(const dp_attn_geom *cg, int dtype, const void *q, const void *k,
                                const void *v, void *m, void *l, void *acc, cudaStream_t st) {
    int rc = check(cg);
    if (rc) return rc;
    AG g = make_ag(cg);
    if (g.sk == 0 || g.sq == 0) return DP_OK;
    int grid = grid_for(g.sq * g.H, 8, 16);
    switch (dtype) {
        case DP_F32:
            attn_fwd_update_simt<float><<<grid, 256, 0, st>>>(g, (const float *)q, (const float *)k,
                (const float *)v, (double *)m, (double *)l, (double *)acc);
            break;
        case DP_F64:
            attn_fwd_update_simt<double><<<grid, 256, 0, st>>>(g, (const double *)q,
                (const double *)k, (const double *)v, (double *)m, (double *)l, (double *)acc);
            break;
        case DP_BF16:
            attn_fwd_update_simt<__nv_bfloat16><<<grid, 256, 0, st>>>(g,
                (const __nv_bfloat16 *)q, (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v,
                (float *)m, (float *)l, (float *)acc);
            break;
        default: set_error("attn: dtype %d", dtype); return DP_ERR_INVALID;
    }
    return launch_status("attn_fwd_update_simt");
}

}  // namespace dp

using namespace dp;

extern "C" int dp_attn_finalize(const dp_attn_geom *cg, int dtype, const void *m, const void *l,
                                const void *acc, void *out, void *lse, void *stream) {
    int rc = check(cg);
    if (rc) return rc;
    AG g = make_ag(cg);
    int64_t total = g.sq * g.H * g.D;
    if (total == 0) return DP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int grid = grid_for(total, 256, 16);
    switch (dtype) {
        case DP_F32:
            attn_finalize_k<float><<<grid, 256, 0, st>>>(g, (const double *)m, (const double *)l,
                (const double *)acc, (float *)out, (double *)lse);
            break;
        case DP_F64:
            attn_finalize_k<double><<<grid, 256, 0, st>>>(g, (const double *)m, (const double *)l,
                (const double *)acc, (double *)out, (double *)lse);
            break;
        case DP_BF16:
            attn_finalize_k<__nv_bfloat16><<<grid, 256, 0, st>>>(g, (const float *)m,
                (const float *)l, (const float *)acc, (__nv_bfloat16 *)out, (float *)lse);
            break;
        default: set_error("attn: dtype %d", dtype); return DP_ERR_INVALID;
    }
    return launch_status("dp_attn_finalize");
}

extern "C" int dp_attn_bwd_preprocess(const dp_attn_geom *cg, int dtype, const void *o,
                                      const void *dout, void *delta, void *stream) {
    int rc = check(cg);
    if (rc) return rc;
    AG g = make_ag(cg);
    if (g.sq == 0) return DP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int grid = grid_for(g.sq * g.H, 8, 16);
    switch (dtype) {
        case DP_F32:
            attn_delta_k<float><<<grid, 256, 0, st>>>(g, (const float *)o, (const float *)dout,
                                                     (double *)delta);
            break;
        case DP_F64:
            attn_delta_k<double><<<grid, 256, 0, st>>>(g, (const double *)o, (const double *)dout,
                                                      (double *)delta);
            break;
        case DP_BF16:
            attn_delta_k<__nv_bfloat16><<<grid, 256, 0, st>>>(g, (const __nv_bfloat16 *)o,
                (const __nv_bfloat16 *)dout, (float *)delta);
            break;
        default: set_error("attn: dtype %d", dtype); return DP_ERR_INVALID;
    }
    return launch_status("dp_attn_bwd_preprocess");
}

namespace dp {
int attn_bwd_update_simt_launch(const dp_attn_geom *cg, int dtype, const void *q, const void *k,
                                const void *v, const void *dout, const void *lse,
                                const void *delta, void *dq, void *dk, void *dv, cudaStream_t st) {
    int rc = check(cg);
    if (rc) return rc;
    AG g = make_ag(cg);
    if (g.sq == 0 || g.sk == 0) return DP_OK;
    int gq = grid_for(g.sq * g.H, 8, 16);
    int gk = grid_for(g.sk * g.H, 8, 16);
    switch (dtype) {
        case DP_F32:
            attn_bwd_dq_simt<float><<<gq, 256, 0, st>>>(g, (const float *)q, (const float *)k,
                (const float *)v, (const float *)dout, (const double *)lse, (const double *)delta,
                (double *)dq);
            attn_bwd_dkdv_simt<float><<<gk, 256, 0, st>>>(g, (const float *)q, (const float *)k,
                (const float *)v, (const float *)dout, (const double *)lse, (const double *)delta,
                (double *)dk, (double *)dv);
            break;
        case DP_F64:
            attn_bwd_dq_simt<double><<<gq, 256, 0, st>>>(g, (const double *)q, (const double *)k,
                (const double *)v, (const double *)dout, (const double *)lse,
                (const double *)delta, (double *)dq);
            attn_bwd_dkdv_simt<double><<<gk, 256, 0, st>>>(g, (const double *)q,
                (const double *)k, (const double *)v, (const double *)dout, (const double *)lse,
                (const double *)delta, (double *)dk, (double *)dv);
            break;
        case DP_BF16:
            attn_bwd_dq_simt<__nv_bfloat16><<<gq, 256, 0, st>>>(g, (const __nv_bfloat16 *)q,
                (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v, (const __nv_bfloat16 *)dout,
                (const float *)lse, (const float *)delta, (float *)dq);
            attn_bwd_dkdv_simt<__nv_bfloat16><<<gk, 256, 0, st>>>(g, (const __nv_bfloat16 *)q,
                (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v, (const __nv_bfloat16 *)dout,
                (const float *)lse, (const float *)delta, (float *)dk, (float *)dv);
            break;
        default: set_error("attn: dtype %d", dtype); return DP_ERR_INVALID;
    }
    return launch_status("attn_bwd_update_simt", 2);
}
}  // namespace dp
