// Register/shared-memory tiled CUDA-core convolution for fp32 / fp64 (the
// reference's dtypes: its fp32 tolerance 1e-5 rules out TF32/bf16 tensor
// math) — stride 1, any spatial rank, any sharded dim with
// the virtual halo block.  The naive per-output kernels in conv_simt.cu
// remain the fallback for strided convolutions.
//
// fwd / dgrad: a CTA owns one output row (b, o0, o1) x 128 positions along
// the last spatial dim x 32 output channels.  Per 8-channel input slab it
// stages the KP*KQ input rows (+KW-1 halo columns, zero-filled from the
// virtual block) and the 8 x taps x 32 weights in shared memory; each thread
// accumulates 4 positions (strided by 32: conflict-free smem reads) x 4
// output channels (one 16-B weight load per tap).  dgrad is the same kernel
// run over the virtual input rows with the flipped, transposed weights read
// in place (W'[ci][co][t] = W[co][ci][T-1-t]).
//
// wgrad: a CTA owns 32 output x 32 input channels and sweeps a share of the
// (row, 64-position) units; thread = (4 output channels, 1 input channel)
// x all taps in registers; per-CTA partials are reduced deterministically.
#include <type_traits>

#include "common.cuh"

namespace dp {
namespace {

// packed fp32x2 FMA (sm_100 FFMA2): two output channels per instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)),
          "l"(*reinterpret_cast<unsigned long long *>(&c)));
    return d;
}

constexpr int kTW = 128;      // fwd positions per CTA
constexpr int kCoT = 32;      // fwd output channels per CTA
constexpr int kCiT = 8;       // fwd input channels per smem slab
constexpr int kWTW = 64;      // wgrad positions per unit
constexpr int kMaxTaps = 27;

struct TG {
    int64_t B, CI, CO;          // kernel's input / output channels
    int64_t in[3], out[3];      // spatial extents (dims aligned right: d2 = last spatial)
    int k[3];
    int64_t base[3];            // window start of output 0 (stride 1)
    int shard;                  // aligned dim with a right halo, or -1
    int64_t halo;
    int64_t xs[5], hs[5];       // input strides (b, c, d0, d1, d2) main / halo block
    int64_t ys[5], y2s[5];      // output strides; rows >= ysplit on dim ysd -> y2
    int ysd;
    int64_t ysplit;
    int flip;                   // dgrad weights
};

// Stage one input row (channel c, spatial v0, v1) columns [v2a, v2a + n) into
// dst with zero fill; lanes of a warp stride over the columns, the row's
// validity / base pointer are computed once.
template <typename T>
__device__ __forceinline__ void async_copy(T *dst, const T *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "n"(sizeof(T))
                 : "memory");
}
__device__ __forceinline__ void async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ void stage_row(const TG &g, const T *__restrict__ x,
                                          const T *__restrict__ xh, int64_t b, int64_t c,
                                          int64_t v0, int64_t v1, int64_t v2a, int n, T *dst,
                                          int lane) {
    bool ok = c < g.CI && v0 >= 0 && v1 >= 0;
    bool hal = false;
    int64_t r0 = v0, r1 = v1;
    if (ok) {
        if (g.shard == 0 && r0 >= g.in[0]) { r0 -= g.in[0]; hal = true; ok = r0 < g.halo; }
        else if (r0 >= g.in[0]) ok = false;
        if (g.shard == 1 && r1 >= g.in[1]) { r1 -= g.in[1]; hal = true; ok = ok && r1 < g.halo; }
        else if (r1 >= g.in[1]) ok = false;
    }
    if (!ok) {
        for (int i = lane; i < n; i += 32) dst[i] = T(0);
        return;
    }
    const T *rowm = x + b * g.xs[0] + c * g.xs[1] + r0 * g.xs[2] + r1 * g.xs[3];
    const T *rowh = xh + b * g.hs[0] + c * g.hs[1] + r0 * g.hs[2] + r1 * g.hs[3];
    const T *row = hal ? rowh : rowm;
    const int64_t st2 = hal ? g.hs[4] : g.xs[4];
    for (int i = lane; i < n; i += 32) {
        int64_t v2 = v2a + i;
        const T *src = nullptr;
        if (v2 >= 0) {
            if (v2 < g.in[2]) src = row + v2 * st2;
            else if (g.shard == 2 && !hal && v2 - g.in[2] < g.halo)
                src = rowh + (v2 - g.in[2]) * g.hs[4];
        }
        // async global -> smem copy: every row of the slab is in flight at once
        // (a load -> store round trip per row serialised the staging on latency)
        if (src) async_copy(dst + i, src);
        else dst[i] = T(0);
    }
}

template <typename T>
__device__ __forceinline__ T fetch_w(const TG &g, const T *__restrict__ w, int64_t co, int64_t ci,
                                     int t, int taps) {
    if (co >= g.CO || ci >= g.CI) return T(0);
    if (!g.flip) return w[(co * g.CI + ci) * taps + t];
    // conv weight [CI(orig c_out)][CO(orig c_in)][taps], flipped taps
    return w[(ci * g.CO + co) * taps + (taps - 1 - t)];
}

template <typename T, int R_, int K2_>   // R_/K2_ = 0: runtime window (else unrolled)
__global__ void __launch_bounds__(256)
conv_tiled_fwd(TG g, const T *__restrict__ x, const T *__restrict__ xh, const T *__restrict__ w,
               T *__restrict__ y, T *__restrict__ y2) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int R = R_ ? R_ : g.k[0] * g.k[1], K2 = K2_ ? K2_ : g.k[2], taps = R * K2;
    const int XW = kTW + K2 - 1;
    T *xs_ = reinterpret_cast<T *>(smraw);                          // [kCiT][R][XW]
    T *ws_ = xs_ + ((kCiT * R * XW + 3) & ~3);                       // [kCiT][taps][kCoT]
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    // decode the output row
    int64_t r = blockIdx.x;
    const int64_t n_wt = (g.out[2] + kTW - 1) / kTW;
    const int64_t wt = r % n_wt; r /= n_wt;
    const int64_t o1 = r % g.out[1]; r /= g.out[1];
    const int64_t o0 = r % g.out[0];
    const int64_t b = r / g.out[0];
    const int64_t ow0 = wt * kTW;
    const int64_t co0 = (int64_t)blockIdx.y * kCoT;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int64_t ci0 = 0; ci0 < g.CI; ci0 += kCiT) {
        for (int rowi = ty; rowi < kCiT * R; rowi += 8) {
            const int cc = rowi / R, rr = rowi % R;
            stage_row<T>(g, x, xh, b, ci0 + cc, g.base[0] + o0 + rr / g.k[1],
                         g.base[1] + o1 + rr % g.k[1], g.base[2] + ow0, XW, xs_ + rowi * XW, tx);
        }
        for (int e = tid; e < kCiT * taps * kCoT; e += 256) {
            const int cc = e / (taps * kCoT), t = (e / kCoT) % taps, c = e % kCoT;
            ws_[e] = fetch_w<T>(g, w, co0 + c, ci0 + cc, t, taps);
        }
        async_wait_all();
        __syncthreads();
#pragma unroll 2
        for (int cc = 0; cc < kCiT; ++cc) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                const T *xr = xs_ + (cc * R + rr) * XW + tx;
                const T *wr = ws_ + (cc * taps + rr * K2) * kCoT + ty * 4;
#pragma unroll
                for (int t2 = 0; t2 < K2; ++t2) {
                    T wv[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) wv[j] = wr[t2 * kCoT + j];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const T xv = xr[32 * i + t2];
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] += xv * wv[j];
                    }
                }
            }
        }
        __syncthreads();
    }
    // store (rows past ysplit on dim ysd go to the halo-gradient block)
    int64_t oo[3] = {o0, o1, 0};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t co = co0 + ty * 4 + j;
        if (co >= g.CO) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t ow = ow0 + tx + 32 * i;
            if (ow >= g.out[2]) continue;
            oo[2] = ow;
            if (g.ysd >= 0 && oo[g.ysd] >= g.ysplit) {
                int64_t q[3] = {oo[0], oo[1], oo[2]};
                q[g.ysd] -= g.ysplit;
                y2[b * g.y2s[0] + co * g.y2s[1] + q[0] * g.y2s[2] + q[1] * g.y2s[3] +
                   q[2] * g.y2s[4]] = acc[i][j];
            } else {
                y[b * g.ys[0] + co * g.ys[1] + oo[0] * g.ys[2] + oo[1] * g.ys[3] +
                  oo[2] * g.ys[4]] = acc[i][j];
            }
        }
    }
}

// wgrad thread = (CPT output channels, 1 input channel); 32 input channels x
// 32 output channels per CTA -> 32 * 32 / CPT threads.
template <typename T, int TMAX, int CPT, int K2_>  // K2_ = 0: runtime
__global__ void __launch_bounds__(32 * 32 / CPT)
conv_tiled_wgrad(TG g, const T *__restrict__ x, const T *__restrict__ xh, const T *__restrict__ dy,
                 T *__restrict__ part, int64_t units, int nbuf) {
    constexpr int kWThreads = 32 * 32 / CPT;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int R = g.k[0] * g.k[1], K2 = K2_ ? K2_ : g.k[2], taps = R * K2;
    const int XW = (kWTW + K2 - 1) | 1;     // odd row length: conflict-free across ci
    T *xs_ = reinterpret_cast<T *>(smraw);  // [32 ci][R][XW]
    // dY tile: [32 co][kWTW], or [kWTW][32 co] (co innermost: 16-B loads of 4
    // output channels) on the fp32 sliding-window path
    constexpr bool kF2 = std::is_same<T, float>::value && K2_ == 3 && TMAX % 3 == 0 && CPT % 4 == 0;
    const int tid = threadIdx.x, cil = tid & 31, cob = tid >> 5;
    const int64_t co0 = (int64_t)blockIdx.y * 32, ci0 = (int64_t)blockIdx.z * 32;
    T acc[kF2 ? 1 : CPT][kF2 ? 1 : TMAX];
    float2 acc2[kF2 ? CPT / 2 : 1][kF2 ? TMAX : 1];
    if constexpr (kF2) {
#pragma unroll
        for (int j = 0; j < CPT / 2; ++j)
#pragma unroll
            for (int t = 0; t < TMAX; ++t) acc2[j][t] = make_float2(0.f, 0.f);
    } else {
#pragma unroll
        for (int j = 0; j < CPT; ++j)
#pragma unroll
            for (int t = 0; t < TMAX; ++t) acc[j][t] = T(0);
    }
    const int64_t n_wt = (g.out[2] + kWTW - 1) / kWTW;
    // two staging buffers: unit k+1 is copied (cp.async) while unit k computes
    const int buf_elems = ((32 * R * XW + 3) & ~3) + 32 * kWTW;
    auto stage = [&](int64_t u, int buf) {
        T *xb = xs_ + (size_t)buf * buf_elems;
        T *db = xb + ((32 * R * XW + 3) & ~3);
        int64_t r = u;
        const int64_t wt = r % n_wt; r /= n_wt;
        const int64_t o1 = r % g.out[1]; r /= g.out[1];
        const int64_t o0 = r % g.out[0];
        const int64_t b = r / g.out[0];
        const int64_t ow0 = wt * kWTW;
        for (int rowi = tid >> 5; rowi < 32 * R; rowi += kWThreads / 32) {
            const int cc = rowi / R, rr = rowi % R;
            stage_row<T>(g, x, xh, b, ci0 + cc, g.base[0] + o0 + rr / g.k[1],
                         g.base[1] + o1 + rr % g.k[1], g.base[2] + ow0, XW, xb + rowi * XW,
                         tid & 31);
        }
        for (int e = tid; e < 32 * kWTW; e += kWThreads) {
            const int cc = e / kWTW, c = e % kWTW;
            const int64_t co = co0 + cc, ow = ow0 + c;
            T *dd = db + (kF2 ? c * 32 + cc : e);
            if (co < g.CO && ow < g.out[2])
                async_copy(dd, dy + b * g.ys[0] + co * g.ys[1] + o0 * g.ys[2] + o1 * g.ys[3] +
                                   ow * g.ys[4]);
            else
                *dd = T(0);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if ((int64_t)blockIdx.x < units) stage(blockIdx.x, 0);
    int buf = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, buf ^= (nbuf - 1)) {
        if (nbuf == 2 && u + gridDim.x < units) {
            stage(u + gridDim.x, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const T *xr = xs_ + (size_t)buf * buf_elems + cil * R * XW;
        T *ds_ = xs_ + (size_t)buf * buf_elems + ((32 * R * XW + 3) & ~3);
        if constexpr (kF2) {
            // fp32: sliding window along the row (each staged input value loaded
            // once per (row r, position), reused by the 3 kw taps), 16-B dY loads,
            // packed fma.rn.f32x2 over output-channel pairs
            constexpr int RM = TMAX / 3;
            float win[RM][3];
#pragma unroll
            for (int rr = 0; rr < RM; ++rr)
                if (rr < R) {
                    win[rr][1] = xr[rr * XW + 0];
                    win[rr][2] = xr[rr * XW + 1];
                }
#pragma unroll 2
            for (int p = 0; p < kWTW; ++p) {
                float2 d2[CPT / 2];
#pragma unroll
                for (int j = 0; j < CPT / 4; ++j) {
                    const float4 v = *reinterpret_cast<const float4 *>(
                        reinterpret_cast<const float *>(ds_) + p * 32 + cob * CPT + 4 * j);
                    d2[2 * j] = make_float2(v.x, v.y);
                    d2[2 * j + 1] = make_float2(v.z, v.w);
                }
#pragma unroll
                for (int rr = 0; rr < RM; ++rr) {
                    if (rr < R) {
                        win[rr][0] = win[rr][1];
                        win[rr][1] = win[rr][2];
                        win[rr][2] = xr[rr * XW + p + 2];
#pragma unroll
                        for (int kw = 0; kw < 3; ++kw) {
                            const float2 xv = make_float2(win[rr][kw], win[rr][kw]);
#pragma unroll
                            for (int j = 0; j < CPT / 2; ++j)
                                acc2[j][rr * 3 + kw] = ffma2(d2[j], xv, acc2[j][rr * 3 + kw]);
                        }
                    }
                }
            }
        } else if (K2_ == 3 && TMAX % 3 == 0) {
            // sliding window along the row: each staged input value is loaded once
            // per (row r, position) and reused by the 3 kw taps from registers
            constexpr int RM = TMAX / 3;
            T win[RM][3];
#pragma unroll
            for (int rr = 0; rr < RM; ++rr)
                if (rr < R) {
                    win[rr][1] = xr[rr * XW + 0];
                    win[rr][2] = xr[rr * XW + 1];
                }
#pragma unroll 4
            for (int p = 0; p < kWTW; ++p) {
                T d[CPT];
#pragma unroll
                for (int j = 0; j < CPT; ++j) d[j] = ds_[(cob * CPT + j) * kWTW + p];
#pragma unroll
                for (int rr = 0; rr < RM; ++rr) {
                    if (rr < R) {
                        win[rr][0] = win[rr][1];
                        win[rr][1] = win[rr][2];
                        win[rr][2] = xr[rr * XW + p + 2];
#pragma unroll
                        for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                            for (int j = 0; j < CPT; ++j) acc[j][rr * 3 + kw] += d[j] * win[rr][kw];
                    }
                }
            }
        } else {
            for (int p = 0; p < kWTW; ++p) {
                T d[CPT];
#pragma unroll
                for (int j = 0; j < CPT; ++j) d[j] = ds_[(cob * CPT + j) * kWTW + p];
#pragma unroll
                for (int t = 0; t < TMAX; ++t) {
                    if (t < taps) {
                        const T xv = xr[(t / K2) * XW + p + t % K2];
#pragma unroll
                        for (int j = 0; j < CPT; ++j) acc[j][t] += d[j] * xv;
                    }
                }
            }
        }
        __syncthreads();
        if (nbuf == 1 && u + gridDim.x < units) stage(u + gridDim.x, 0);
    }
    // partial [blockIdx.x][co][ci][taps]
    const int64_t ci = ci0 + cil;
    if (ci >= g.CI) return;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        const int64_t co = co0 + cob * CPT + j;
        if (co >= g.CO) continue;
        T *dst = part + (((int64_t)blockIdx.x * g.CO + co) * g.CI + ci) * taps;
#pragma unroll
        for (int t = 0; t < TMAX; ++t)
            if (t < taps) {
                if constexpr (kF2)
                    dst[t] = (j & 1) ? acc2[j / 2][t].y : acc2[j / 2][t].x;
                else
                    dst[t] = acc[j][t];
            }
    }
}

template <typename T>
__global__ void tiled_wgrad_reduce(const T *__restrict__ part, T *__restrict__ dw, int64_t n,
                                   int chunks) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        T s = T(0);
        for (int c = 0; c < chunks; ++c) s += part[c * n + i];
        dw[i] = s;
    }
}

// Right-align the spatial dims (last spatial -> index 2) of a dp_conv_geom.
void align3(const dp_conv_geom *cg, int64_t *in, int64_t *out, int *k, int64_t *base, int *shard,
            int64_t *xs, int64_t *hs, int64_t *ys) {
    const int off = 3 - cg->nsp;
    for (int i = 0; i < 3; ++i) {
        in[i] = out[i] = 1;
        k[i] = 1;
        base[i] = 0;
        xs[2 + i] = hs[2 + i] = ys[2 + i] = 0;
    }
    xs[0] = cg->xs[0]; xs[1] = cg->xs[1];
    hs[0] = cg->hs[0]; hs[1] = cg->hs[1];
    ys[0] = cg->ys[0]; ys[1] = cg->ys[1];
    for (int i = 0; i < cg->nsp; ++i) {
        in[off + i] = cg->in_ext[i];
        out[off + i] = cg->out_ext[i];
        k[off + i] = cg->kernel[i];
        base[off + i] = cg->base[i];
        xs[2 + off + i] = cg->xs[2 + i];
        hs[2 + off + i] = cg->hs[2 + i];
        ys[2 + off + i] = cg->ys[2 + i];
    }
    *shard = cg->shard >= 0 ? cg->shard + off : -1;
}

size_t fwd_smem(const TG &g, int es) {
    const int R = g.k[0] * g.k[1], taps = R * g.k[2];
    const size_t xn = ((size_t)kCiT * R * (kTW + g.k[2] - 1) + 3) & ~(size_t)3;
    return (xn + (size_t)kCiT * taps * kCoT) * es;
}
size_t wgrad_smem(const TG &g, int es) {
    const int R = g.k[0] * g.k[1];
    const int XW = (kWTW + g.k[2] - 1) | 1;
    const size_t one = ((((size_t)32 * R * XW + 3) & ~(size_t)3) + 32 * kWTW) * es;
    return 2 * one <= 200 * 1024 ? 2 * one : one;   // double-buffered when it fits
}

template <typename T>
int launch_fwd(const TG &g, const void *x, const void *xh, const void *w, void *y, void *y2,
               cudaStream_t st) {
    const int64_t rows = g.B * g.out[0] * g.out[1] * ((g.out[2] + kTW - 1) / kTW);
    if (rows == 0) return DP_OK;
    DP_REQUIRE(rows < (1ll << 31), DP_ERR_UNSUPPORTED, "conv_tiled: grid too large");
    const size_t smem = fwd_smem(g, sizeof(T));
    dim3 grid((unsigned)rows, (unsigned)((g.CO + kCoT - 1) / kCoT));
    const int R = g.k[0] * g.k[1], K2 = g.k[2];
    auto kern = (R == 3 && K2 == 3)   ? conv_tiled_fwd<T, 3, 3>
                : (R == 9 && K2 == 3) ? conv_tiled_fwd<T, 9, 3>
                : (R == 1 && K2 == 3) ? conv_tiled_fwd<T, 1, 3>
                                      : conv_tiled_fwd<T, 0, 0>;
    DP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 256, smem, st>>>(g, (const T *)x, (const T *)xh, (const T *)w, (T *)y,
                                  (T *)(y2 ? y2 : y));
    return launch_status("conv_tiled_fwd");
}

bool tiled_ok(const dp_conv_geom *cg, int dtype) {
    if (dtype != DP_F32 && dtype != DP_F64) return false;
    for (int i = 0; i < cg->nsp; ++i)
        if (cg->stride[i] != 1) return false;
    int taps = 1, rows = 1;
    for (int i = 0; i < cg->nsp; ++i) taps *= cg->kernel[i];
    for (int i = 0; i + 1 < cg->nsp; ++i) rows *= cg->kernel[i];
    if (taps > kMaxTaps || cg->kernel[cg->nsp - 1] > 15) return false;
    return rows * (kWTW + 15) * 32 * 8 + 32 * kWTW * 8 <= 200 * 1024;
}

}  // namespace

int conv_tiled_eligible(const dp_conv_geom *cg, int dtype) { return tiled_ok(cg, dtype) ? 1 : 0; }

int conv_fwd_tiled_launch(const dp_conv_geom *cg, int dtype, const void *x, const void *xh,
                          const void *w, void *y, cudaStream_t st) {
    TG g;
    memset(&g, 0, sizeof(g));
    g.B = cg->batch;
    g.CI = cg->c_in;
    g.CO = cg->c_out;
    align3(cg, g.in, g.out, g.k, g.base, &g.shard, g.xs, g.hs, g.ys);
    g.halo = cg->halo;
    if (g.halo == 0) g.shard = -1;
    g.ysd = -1;
    g.flip = 0;
    return dtype == DP_F64 ? launch_fwd<double>(g, x, xh, w, y, nullptr, st)
                           : launch_fwd<float>(g, x, xh, w, y, nullptr, st);
}

// dgrad of a stride-1 conv = forward conv of dy over the virtual input rows
// [0, in + halo) with base' = -(base + k - 1) and flipped, transposed weights.
int conv_dgrad_tiled_launch(const dp_conv_geom *cg, int dtype, const void *dy, const void *w,
                            void *dx, void *dxh, cudaStream_t st) {
    int64_t in[3], out[3], base[3], xs[5], hs[5], ys[5];
    int k[3], shard;
    align3(cg, in, out, k, base, &shard, xs, hs, ys);
    TG g;
    memset(&g, 0, sizeof(g));
    g.B = cg->batch;
    g.CI = cg->c_out;   // dy channels
    g.CO = cg->c_in;    // dx channels
    for (int i = 0; i < 3; ++i) {
        g.in[i] = out[i];                       // dy extents
        g.out[i] = in[i] + (i == shard ? cg->halo : 0);
        g.k[i] = k[i];
        g.base[i] = -(base[i] + k[i] - 1);
    }
    g.shard = -1;
    g.halo = 0;
    for (int i = 0; i < 5; ++i) {
        g.xs[i] = ys[i];
        g.hs[i] = ys[i];
        g.ys[i] = xs[i];
        g.y2s[i] = hs[i];
    }
    g.ysd = (shard >= 0 && cg->halo > 0) ? shard : -1;
    g.ysplit = shard >= 0 ? in[shard] : 0;
    g.flip = 1;
    return dtype == DP_F64 ? launch_fwd<double>(g, dy, dy, w, dx, dxh, st)
                           : launch_fwd<float>(g, dy, dy, w, dx, dxh, st);
}

static TG wgrad_geom(const dp_conv_geom *cg) {
    TG g;
    memset(&g, 0, sizeof(g));
    g.B = cg->batch;
    g.CI = cg->c_in;
    g.CO = cg->c_out;
    align3(cg, g.in, g.out, g.k, g.base, &g.shard, g.xs, g.hs, g.ys);
    g.halo = cg->halo;
    if (g.halo == 0) g.shard = -1;
    g.ysd = -1;
    return g;
}

static int wgrad_chunks_tiled(const TG &g, int64_t units) {
    const int64_t tiles = ((g.CO + 31) / 32) * ((g.CI + 31) / 32);
    int64_t want = (6 * sm_count() + tiles - 1) / tiles;   // several CTAs per SM hide staging
    if (want > units) want = units;
    return (int)(want < 1 ? 1 : want);
}

int64_t conv_wgrad_tiled_workspace(const dp_conv_geom *cg, int dtype) {
    TG g = wgrad_geom(cg);
    const int64_t units = g.B * g.out[0] * g.out[1] * ((g.out[2] + kWTW - 1) / kWTW);
    const int64_t taps = (int64_t)g.k[0] * g.k[1] * g.k[2];
    return (int64_t)wgrad_chunks_tiled(g, units) * g.CO * g.CI * taps * (dtype == DP_F64 ? 8 : 4);
}

int conv_wgrad_tiled_launch(const dp_conv_geom *cg, int dtype, const void *x, const void *xh,
                            const void *dy, void *dw, void *ws, int64_t ws_bytes, cudaStream_t st) {
    TG g = wgrad_geom(cg);
    const int64_t units = g.B * g.out[0] * g.out[1] * ((g.out[2] + kWTW - 1) / kWTW);
    const int taps = g.k[0] * g.k[1] * g.k[2];
    const int64_t n = g.CO * g.CI * taps;
    const int es = dtype == DP_F64 ? 8 : 4;
    if (units == 0) {
        DP_CUDA_CHECK(cudaMemsetAsync(dw, 0, n * es, st));
        return DP_OK;
    }
    const int chunks = wgrad_chunks_tiled(g, units);
    DP_REQUIRE(ws_bytes >= (int64_t)chunks * n * es, DP_ERR_INVALID,
               "conv_wgrad_tiled: workspace too small");
    const size_t smem = wgrad_smem(g, es);
    const int R = g.k[0] * g.k[1];
    const size_t one = ((((size_t)32 * R * ((kWTW + g.k[2] - 1) | 1) + 3) & ~(size_t)3) +
                        32 * kWTW) * es;
    const int nbuf = smem >= 2 * one ? 2 : 1;
    dim3 grid((unsigned)chunks, (unsigned)((g.CO + 31) / 32), (unsigned)((g.CI + 31) / 32));
    const int rgrid = grid_for(n, 256, 4);
    const bool small = taps <= 9;
#define DP_TW(T, TM, CP)                                                                          \
    do {                                                                                          \
        auto kern = g.k[2] == 3 ? conv_tiled_wgrad<T, TM, CP, 3> : conv_tiled_wgrad<T, TM, CP, 0>; \
        DP_CUDA_CHECK(cudaFuncSetAttribute(kern,                                                  \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        kern<<<grid, 32 * 32 / CP, smem, st>>>(                                                   \
            g, (const T *)x, (const T *)xh, (const T *)dy, (T *)ws, units, nbuf);                 \
        tiled_wgrad_reduce<T><<<rgrid, 256, 0, st>>>((const T *)ws, (T *)dw, n, chunks);          \
    } while (0)
    if (dtype == DP_F64) {
        if (small) DP_TW(double, 9, 8);
        else DP_TW(double, kMaxTaps, 4);
    } else {
        if (small) DP_TW(float, 9, 8);
        else DP_TW(float, kMaxTaps, 4);
    }
#undef DP_TW
    return launch_status("conv_tiled_wgrad", 2);
}

}  // namespace dp
