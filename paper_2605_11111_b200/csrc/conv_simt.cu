// Direct (CUDA-core) convolution kernels over the virtual halo block.
//
// These cover the whole envelope the reference supports — 1-D/2-D (and
// 3-D) spatial dims, any odd kernel, any stride/padding, any sharded
// spatial dim, batched or not, any strides/layout — in fp32, fp64 and bf16
// (fp32 accumulate).  The tcgen05 implicit-GEMM kernels (conv_tc.cu) take
// over for the large bf16 channels-last stride-1 cases; these are the
// general path and the fp32/fp64 parity path (reference fp32 tolerance
// 1e-5 rules out TF32/bf16 tensor math for fp32 inputs).
//
// Virtual indexing (dp_conv_geom): output o of spatial dim i reads virtual
// rows base[i] + o*stride[i] + t.  On the sharded dim, rows [0, in_ext)
// come from the main block and [in_ext, in_ext + halo) from the halo
// block; all other rows are zero.  This reproduces domainpar/ops.py:397-413
// (trim + np.pad + dense.conv with the sharded padding materialised).
#include "common.cuh"

namespace dp {
namespace {

struct Geo {
    int nsp, shard;
    int64_t B, Ci, Co;
    int64_t in[3], out[3], halo;
    int k[3], s[3];
    int64_t base[3];
    int64_t xs[5], hs[5], ys[5];
};

Geo make_geo(const dp_conv_geom *g) {
    Geo o;
    o.nsp = g->nsp;
    o.shard = g->shard;
    o.B = g->batch;
    o.Ci = g->c_in;
    o.Co = g->c_out;
    o.halo = g->halo;
    for (int i = 0; i < 3; ++i) {
        bool live = i < g->nsp;
        o.in[i] = live ? g->in_ext[i] : 1;
        o.out[i] = live ? g->out_ext[i] : 1;
        o.k[i] = live ? g->kernel[i] : 1;
        o.s[i] = live ? g->stride[i] : 1;
        o.base[i] = live ? g->base[i] : 0;
    }
    for (int i = 0; i < 5; ++i) {
        o.xs[i] = (i < 2 + g->nsp) ? g->xs[i] : 0;
        o.hs[i] = (i < 2 + g->nsp) ? g->hs[i] : 0;
        o.ys[i] = (i < 2 + g->nsp) ? g->ys[i] : 0;
    }
    return o;
}

// Pointer offset of virtual input (b, c, v0, v1, v2); -1 when it is a zero.
// `in_halo` tells which tensor the offset refers to.
__device__ __forceinline__ int64_t vin_offset(const Geo &g, int64_t b, int64_t c, const int64_t *v,
                                               bool &in_halo) {
    in_halo = false;
    int64_t off_main = b * g.xs[0] + c * g.xs[1];
    int64_t off_halo = b * g.hs[0] + c * g.hs[1];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        int64_t vi = v[i];
        if (vi < 0) return -1;
        if (i == g.shard && vi >= g.in[i]) {
            vi -= g.in[i];
            if (vi >= g.halo) return -1;
            in_halo = true;
            off_halo += vi * g.hs[2 + i];
            off_main += 0;
        } else {
            if (vi >= g.in[i]) return -1;
            off_main += vi * g.xs[2 + i];
            off_halo += vi * g.hs[2 + i];
        }
    }
    return in_halo ? off_halo : off_main;
}

// ---- forward: one thread per output element --------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
conv_fwd_simt(Geo g, const T *__restrict__ x, const T *__restrict__ xh, const T *__restrict__ w,
              T *__restrict__ y) {
    using A = typename Acc<T>::type;
    const int64_t total = g.B * g.Co * g.out[0] * g.out[1] * g.out[2];
    const int taps = g.k[0] * g.k[1] * g.k[2];
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx;
        int64_t o2 = r % g.out[2]; r /= g.out[2];
        int64_t o1 = r % g.out[1]; r /= g.out[1];
        int64_t o0 = r % g.out[0]; r /= g.out[0];
        int64_t co = r % g.Co;
        int64_t b = r / g.Co;
        A acc = 0;
        const T *wc = w + co * g.Ci * taps;
        for (int64_t ci = 0; ci < g.Ci; ++ci) {
            for (int t0 = 0; t0 < g.k[0]; ++t0) {
                for (int t1 = 0; t1 < g.k[1]; ++t1) {
                    for (int t2 = 0; t2 < g.k[2]; ++t2) {
                        int64_t v[3] = {g.base[0] + o0 * g.s[0] + t0, g.base[1] + o1 * g.s[1] + t1,
                                        g.base[2] + o2 * g.s[2] + t2};
                        bool hal;
                        int64_t off = vin_offset(g, b, ci, v, hal);
                        if (off < 0) continue;
                        A xv = to_acc(hal ? xh[off] : x[off]);
                        A wv = to_acc(wc[(ci * g.k[0] + t0) * g.k[1] * g.k[2] + t1 * g.k[2] + t2]);
                        acc += xv * wv;
                    }
                }
            }
        }
        y[b * g.ys[0] + co * g.ys[1] + o0 * g.ys[2] + o1 * g.ys[3] + o2 * g.ys[4]] = from_acc<T>(acc);
    }
}

// ---- dgrad: one thread per virtual input element ---------------------------
template <typename T>
__global__ void __launch_bounds__(256)
conv_dgrad_simt(Geo g, const T *__restrict__ dy, const T *__restrict__ w, T *__restrict__ dx,
                T *__restrict__ dxh) {
    using A = typename Acc<T>::type;
    int64_t vext[3] = {g.in[0], g.in[1], g.in[2]};
    if (g.shard >= 0) vext[g.shard] += g.halo;
    const int64_t total = g.B * g.Ci * vext[0] * vext[1] * vext[2];
    const int taps = g.k[0] * g.k[1] * g.k[2];
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx;
        int64_t v2 = r % vext[2]; r /= vext[2];
        int64_t v1 = r % vext[1]; r /= vext[1];
        int64_t v0 = r % vext[0]; r /= vext[0];
        int64_t ci = r % g.Ci;
        int64_t b = r / g.Ci;
        int64_t v[3] = {v0, v1, v2};
        A acc = 0;
        for (int t0 = 0; t0 < g.k[0]; ++t0) {
            int64_t n0 = v[0] - g.base[0] - t0;
            if (n0 < 0 || n0 % g.s[0]) continue;
            int64_t o0 = n0 / g.s[0];
            if (o0 >= g.out[0]) continue;
            for (int t1 = 0; t1 < g.k[1]; ++t1) {
                int64_t n1 = v[1] - g.base[1] - t1;
                if (n1 < 0 || n1 % g.s[1]) continue;
                int64_t o1 = n1 / g.s[1];
                if (o1 >= g.out[1]) continue;
                for (int t2 = 0; t2 < g.k[2]; ++t2) {
                    int64_t n2 = v[2] - g.base[2] - t2;
                    if (n2 < 0 || n2 % g.s[2]) continue;
                    int64_t o2 = n2 / g.s[2];
                    if (o2 >= g.out[2]) continue;
                    const T *dyp = dy + b * g.ys[0] + o0 * g.ys[2] + o1 * g.ys[3] + o2 * g.ys[4];
                    const int tap = (t0 * g.k[1] + t1) * g.k[2] + t2;
                    for (int64_t co = 0; co < g.Co; ++co)
                        acc += to_acc(dyp[co * g.ys[1]]) * to_acc(w[(co * g.Ci + ci) * taps + tap]);
                }
            }
        }
        bool halo_row = g.shard >= 0 && v[g.shard] >= g.in[g.shard];
        if (halo_row) {
            int64_t vv[3] = {v0, v1, v2};
            vv[g.shard] -= g.in[g.shard];
            dxh[b * g.hs[0] + ci * g.hs[1] + vv[0] * g.hs[2] + vv[1] * g.hs[3] + vv[2] * g.hs[4]] =
                from_acc<T>(acc);
        } else {
            dx[b * g.xs[0] + ci * g.xs[1] + v0 * g.xs[2] + v1 * g.xs[3] + v2 * g.xs[4]] =
                from_acc<T>(acc);
        }
    }
}

// ---- wgrad: split-K partials + deterministic reduction ---------------------
constexpr int kTapGroup = 32;

template <typename T>
__global__ void __launch_bounds__(256)
conv_wgrad_partial(Geo g, const T *__restrict__ x, const T *__restrict__ xh,
                   const T *__restrict__ dy, typename Acc<T>::type *__restrict__ part,
                   int64_t chunk, int tap_groups) {
    using A = typename Acc<T>::type;
    __shared__ A red[8][kTapGroup];
    const int taps = g.k[0] * g.k[1] * g.k[2];
    const int64_t co = blockIdx.z, ci = blockIdx.y;
    const int tg = blockIdx.x % tap_groups;
    const int64_t ch = blockIdx.x / tap_groups;
    const int t_lo = tg * kTapGroup;
    const int nt = min(kTapGroup, taps - t_lo);
    const int64_t npos = g.B * g.out[0] * g.out[1] * g.out[2];
    const int64_t p_lo = ch * chunk, p_hi = min(npos, p_lo + chunk);
    A acc[kTapGroup];
#pragma unroll
    for (int t = 0; t < kTapGroup; ++t) acc[t] = 0;
    for (int64_t p = p_lo + threadIdx.x; p < p_hi; p += blockDim.x) {
        int64_t r = p;
        int64_t o2 = r % g.out[2]; r /= g.out[2];
        int64_t o1 = r % g.out[1]; r /= g.out[1];
        int64_t o0 = r % g.out[0];
        int64_t b = r / g.out[0];
        A d = to_acc(dy[b * g.ys[0] + co * g.ys[1] + o0 * g.ys[2] + o1 * g.ys[3] + o2 * g.ys[4]]);
#pragma unroll
        for (int t = 0; t < kTapGroup; ++t) {
            if (t < nt) {
                int tap = t_lo + t;
                int t2 = tap % g.k[2];
                int t1 = (tap / g.k[2]) % g.k[1];
                int t0 = tap / (g.k[2] * g.k[1]);
                int64_t v[3] = {g.base[0] + o0 * g.s[0] + t0, g.base[1] + o1 * g.s[1] + t1,
                                g.base[2] + o2 * g.s[2] + t2};
                bool hal;
                int64_t off = vin_offset(g, b, ci, v, hal);
                if (off >= 0) acc[t] += d * to_acc(hal ? xh[off] : x[off]);
            }
        }
    }
    // block reduction: warp shuffle, then across the 8 warps
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < kTapGroup; ++t) {
        A v = acc[t];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[wid][t] = v;
    }
    __syncthreads();
    if (threadIdx.x < nt) {
        A v = 0;
        for (int i = 0; i < 8; ++i) v += red[i][threadIdx.x];
        part[((ch * g.Co + co) * g.Ci + ci) * taps + t_lo + threadIdx.x] = v;
    }
}

template <typename A>
__global__ void wgrad_reduce(const A *__restrict__ part, A *__restrict__ dw, int64_t n, int64_t chunks) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        A s = 0;
        for (int64_t c = 0; c < chunks; ++c) s += part[c * n + i];
        dw[i] = s;
    }
}

int64_t wgrad_chunks(const Geo &g) {
    const int64_t npos = g.B * g.out[0] * g.out[1] * g.out[2];
    // aim for a few thousand blocks in total, >= 4096 positions per block
    int64_t pairs = g.Co * g.Ci;
    int64_t want = (4 * sm_count() * 8 + pairs - 1) / pairs;
    int64_t by_size = (npos + 4095) / 4096;
    int64_t c = want < by_size ? want : by_size;
    return c < 1 ? 1 : c;
}

int check_geom(const dp_conv_geom *g) {
    DP_REQUIRE(g, DP_ERR_INVALID, "conv: null geometry");
    DP_REQUIRE(g->nsp >= 1 && g->nsp <= 3, DP_ERR_INVALID, "conv: nsp %d", g->nsp);
    DP_REQUIRE(g->shard >= -1 && g->shard < g->nsp, DP_ERR_INVALID, "conv: shard %d", g->shard);
    DP_REQUIRE(g->batch >= 0 && g->c_in >= 1 && g->c_out >= 1, DP_ERR_INVALID, "conv: B/C");
    for (int i = 0; i < g->nsp; ++i) {
        DP_REQUIRE(g->kernel[i] >= 1 && g->stride[i] >= 1, DP_ERR_INVALID, "conv: kernel/stride");
        DP_REQUIRE(g->out_ext[i] >= 0 && g->in_ext[i] >= 0, DP_ERR_INVALID, "conv: extents");
    }
    return DP_OK;
}

}  // namespace

// tiled fp32/fp64 kernels (conv_tiled.cu) for stride-1 convolutions
int conv_tiled_eligible(const dp_conv_geom *, int dtype);
int conv_fwd_tiled_launch(const dp_conv_geom *, int, const void *, const void *, const void *,
                          void *, cudaStream_t);
int conv_dgrad_tiled_launch(const dp_conv_geom *, int, const void *, const void *, void *, void *,
                            cudaStream_t);
int64_t conv_wgrad_tiled_workspace(const dp_conv_geom *, int);
int conv_wgrad_tiled_launch(const dp_conv_geom *, int, const void *, const void *, const void *,
                            void *, void *, int64_t, cudaStream_t);

// entry points used by capi (conv_tc.cu decides between TC and these)
int conv_fwd_simt_launch(const dp_conv_geom *cg, int dtype, const void *x, const void *xh,
                         const void *w, void *y, cudaStream_t st) {
    int rc = check_geom(cg);
    if (rc) return rc;
    if (conv_tiled_eligible(cg, dtype)) return conv_fwd_tiled_launch(cg, dtype, x, xh, w, y, st);
    Geo g = make_geo(cg);
    int64_t total = g.B * g.Co * g.out[0] * g.out[1] * g.out[2];
    if (total == 0) return DP_OK;
    int grid = grid_for(total, 256, 16);
    switch (dtype) {
        case DP_F32:
            conv_fwd_simt<float><<<grid, 256, 0, st>>>(g, (const float *)x, (const float *)xh,
                                                      (const float *)w, (float *)y);
            break;
        case DP_F64:
            conv_fwd_simt<double><<<grid, 256, 0, st>>>(g, (const double *)x, (const double *)xh,
                                                       (const double *)w, (double *)y);
            break;
        case DP_BF16:
            conv_fwd_simt<__nv_bfloat16><<<grid, 256, 0, st>>>(
                g, (const __nv_bfloat16 *)x, (const __nv_bfloat16 *)xh,
                (const __nv_bfloat16 *)w, (__nv_bfloat16 *)y);
            break;
        default:
            set_error("conv: dtype %d", dtype);
            return DP_ERR_INVALID;
    }
    return launch_status("conv_fwd_simt");
}

int conv_dgrad_simt_launch(const dp_conv_geom *cg, int dtype, const void *dy, const void *w,
                           void *dx, void *dxh, cudaStream_t st) {
    int rc = check_geom(cg);
    if (rc) return rc;
    if (conv_tiled_eligible(cg, dtype)) return conv_dgrad_tiled_launch(cg, dtype, dy, w, dx, dxh, st);
    Geo g = make_geo(cg);
    int64_t vext = 1;
    for (int i = 0; i < 3; ++i) vext *= g.in[i] + (i == g.shard ? g.halo : 0);
    int64_t total = g.B * g.Ci * vext;
    if (total == 0) return DP_OK;
    int grid = grid_for(total, 256, 16);
    switch (dtype) {
        case DP_F32:
            conv_dgrad_simt<float><<<grid, 256, 0, st>>>(g, (const float *)dy, (const float *)w,
                                                        (float *)dx, (float *)dxh);
            break;
        case DP_F64:
            conv_dgrad_simt<double><<<grid, 256, 0, st>>>(g, (const double *)dy, (const double *)w,
                                                         (double *)dx, (double *)dxh);
            break;
        case DP_BF16:
            conv_dgrad_simt<__nv_bfloat16><<<grid, 256, 0, st>>>(
                g, (const __nv_bfloat16 *)dy, (const __nv_bfloat16 *)w, (__nv_bfloat16 *)dx,
                (__nv_bfloat16 *)dxh);
            break;
        default:
            set_error("conv: dtype %d", dtype);
            return DP_ERR_INVALID;
    }
    return launch_status("conv_dgrad_simt");
}

int64_t conv_wgrad_simt_workspace(const dp_conv_geom *cg, int dtype) {
    if (conv_tiled_eligible(cg, dtype)) return conv_wgrad_tiled_workspace(cg, dtype);
    Geo g = make_geo(cg);
    int64_t taps = (int64_t)g.k[0] * g.k[1] * g.k[2];
    int64_t el = dtype == DP_F64 ? 8 : 4;
    return wgrad_chunks(g) * g.Co * g.Ci * taps * el;
}

int conv_wgrad_simt_launch(const dp_conv_geom *cg, int dtype, const void *x, const void *xh,
                           const void *dy, void *dw, void *ws, int64_t ws_bytes, cudaStream_t st) {
    int rc = check_geom(cg);
    if (rc) return rc;
    if (conv_tiled_eligible(cg, dtype))
        return conv_wgrad_tiled_launch(cg, dtype, x, xh, dy, dw, ws, ws_bytes, st);
    Geo g = make_geo(cg);
    const int taps = g.k[0] * g.k[1] * g.k[2];
    const int64_t n = g.Co * g.Ci * taps;
    const int64_t npos = g.B * g.out[0] * g.out[1] * g.out[2];
    const int el = dtype == DP_F64 ? 8 : 4;
    if (npos == 0) {
        DP_CUDA_CHECK(cudaMemsetAsync(dw, 0, n * el, st));
        return DP_OK;
    }
    const int64_t chunks = wgrad_chunks(g);
    DP_REQUIRE(ws_bytes >= chunks * n * el, DP_ERR_INVALID, "conv_wgrad: workspace too small");
    const int64_t chunk = (npos + chunks - 1) / chunks;
    const int tap_groups = (taps + kTapGroup - 1) / kTapGroup;
    dim3 grid((unsigned)(chunks * tap_groups), (unsigned)g.Ci, (unsigned)g.Co);
    DP_REQUIRE(g.Ci < 65536 && g.Co < 65536, DP_ERR_UNSUPPORTED, "conv_wgrad: channels");
    int rgrid = grid_for(n, 256, 4);
    switch (dtype) {
        case DP_F32:
            conv_wgrad_partial<float><<<grid, 256, 0, st>>>(g, (const float *)x, (const float *)xh,
                                                           (const float *)dy, (float *)ws, chunk,
                                                           tap_groups);
            wgrad_reduce<float><<<rgrid, 256, 0, st>>>((const float *)ws, (float *)dw, n, chunks);
            break;
        case DP_F64:
            conv_wgrad_partial<double><<<grid, 256, 0, st>>>(
                g, (const double *)x, (const double *)xh, (const double *)dy, (double *)ws, chunk,
                tap_groups);
            wgrad_reduce<double><<<rgrid, 256, 0, st>>>((const double *)ws, (double *)dw, n, chunks);
            break;
        case DP_BF16:
            conv_wgrad_partial<__nv_bfloat16><<<grid, 256, 0, st>>>(
                g, (const __nv_bfloat16 *)x, (const __nv_bfloat16 *)xh,
                (const __nv_bfloat16 *)dy, (float *)ws, chunk, tap_groups);
            wgrad_reduce<float><<<rgrid, 256, 0, st>>>((const float *)ws, (float *)dw, n, chunks);
            break;
        default:
            set_error("conv: dtype %d", dtype);
            return DP_ERR_INVALID;
    }
    return launch_status("conv_wgrad_simt", 2);
}

}  // namespace dp
