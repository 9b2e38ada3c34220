// Sharded normalisations and pointwise ops:
//   sharded_layer_norm  domainpar/ops.py:153-173  (fp64 moments, ONE stacked all_reduce)
//   sharded_softmax     domainpar/ops.py:126-150  (all_reduce max, then all_reduce sum)
//   dense.softmax / dense.layer_norm  domainpar/dense.py:223-255 (the unsharded case)
//   sharded_elementwise domainpar/ops.py:93-104 + dense.py:65-98 (add / mul / scale)
//
// The reduced dim is viewed as [outer, n, inner] with element strides.  Stats
// accumulate in fp64 (the reference's float64 statistics), in a deterministic
// order: per-(o, i) partials over fixed n-chunks, then a fixed-order combine
// (bitwise-reproducible, no atomics).  The host all-reduces the combined
// stats between the passes (one NCCL call: both layer-norm moments ride one
// buffer, as dp/ops.py:168).  Pointwise math runs in fp64 for fp64 tensors
// and fp32 otherwise (the reference's fp64 exp of an fp32 input differs
// from expf by < 1e-7 relative, far inside its fp32 tolerance of 1e-5).
// All kernels are HBM-bound: one read of x for the stats, one read + one
// write for the apply pass.
#include "common.cuh"

namespace dp {
namespace {

template <typename T> struct Pw { using type = float; };
template <> struct Pw<double> { using type = double; };

__device__ __forceinline__ double ld64(const float *p) { return (double)*p; }
__device__ __forceinline__ double ld64(const double *p) { return *p; }
__device__ __forceinline__ double ld64(const __nv_bfloat16 *p) { return (double)__bfloat162float(*p); }

__device__ __forceinline__ float pw_exp(float v) { return expf(v); }
__device__ __forceinline__ double pw_exp(double v) { return exp(v); }

struct View3 {
    int64_t outer, n, inner;
    int64_t so, sn, si;   // element strides
};

// kind: 0 moments (s1, s2), 1 max, 2 sum exp(x - aux)
template <typename T, int KIND>
__global__ void stats_partial(View3 v, const T *__restrict__ x, const double *__restrict__ aux,
                              double *__restrict__ part, int64_t chunk, int nsplit) {
    const int64_t cells = v.outer * v.inner;
    if (v.inner == 1) {
        // warp per (row, chunk): lanes stride along n (contiguous when sn == 1)
        const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
        const int lane = threadIdx.x & 31;
        for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
             w < cells * nsplit; w += warps) {
            const int64_t o = w % cells, sp = w / cells;
            const int64_t j0 = sp * chunk, j1 = min(v.n, j0 + chunk);
            const T *row = x + o * v.so;
            double a = KIND == 1 ? -INFINITY : 0.0, b = 0.0;
            const double m = KIND == 2 ? aux[o] : 0.0;
            for (int64_t j = j0 + lane; j < j1; j += 32) {
                const double xv = ld64(row + j * v.sn);
                if (KIND == 0) {
                    a += xv;
                    b += xv * xv;
                } else if (KIND == 1) {
                    a = fmax(a, xv);
                } else {
                    using P = typename Pw<T>::type;
                    a += (double)pw_exp((P)(xv - m));
                }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const double oa = __shfl_xor_sync(0xffffffffu, a, off);
                if (KIND == 1) a = fmax(a, oa); else a += oa;
                if (KIND == 0) b += __shfl_xor_sync(0xffffffffu, b, off);
            }
            if (lane == 0) {
                part[sp * cells + o] = a;
                if (KIND == 0) part[(int64_t)(nsplit + sp) * cells + o] = b;
            }
        }
        return;
    }
    // thread per (o, i) and chunk: consecutive threads read consecutive i
    const int64_t total = cells * nsplit;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t % cells, sp = t / cells;
        const int64_t o = c / v.inner, i = c % v.inner;
        const int64_t j0 = sp * chunk, j1 = min(v.n, j0 + chunk);
        const T *col = x + o * v.so + i * v.si;
        double a = KIND == 1 ? -INFINITY : 0.0, b = 0.0;
        const double m = KIND == 2 ? aux[c] : 0.0;
        for (int64_t j = j0; j < j1; ++j) {
            const double xv = ld64(col + j * v.sn);
            if (KIND == 0) {
                a += xv;
                b += xv * xv;
            } else if (KIND == 1) {
                a = fmax(a, xv);
            } else {
                using P = typename Pw<T>::type;
                a += (double)pw_exp((P)(xv - m));
            }
        }
        part[sp * cells + c] = a;
        if (KIND == 0) part[(int64_t)(nsplit + sp) * cells + c] = b;
    }
}

// fixed-order combine of the split partials -> stats [nstat][cells]
__global__ void stats_combine(const double *__restrict__ part, double *__restrict__ stats,
                              int64_t cells, int nsplit, int nstat, int is_max) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells * nstat;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = c / cells, cc = c % cells;
        const double *p = part + s * nsplit * cells + cc;
        double a = is_max ? -INFINITY : 0.0;
        for (int k = 0; k < nsplit; ++k) a = is_max ? fmax(a, p[k * cells]) : a + p[k * cells];
        stats[c] = a;
    }
}

// layer norm: stats = global (s1, s2); softmax: stats = global denom, aux = global max
template <typename T, int KIND>
__global__ void norm_apply(View3 v, const T *__restrict__ x, T *__restrict__ y, View3 vy,
                           const double *__restrict__ stats, const double *__restrict__ aux,
                           double count, double eps) {
    const int64_t cells = v.outer * v.inner;
    const int64_t total = cells * v.n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % v.inner, r = e / v.inner;
        const int64_t j = r % v.n, o = r / v.n;
        const int64_t c = o * v.inner + i;
        const double xv = ld64(x + o * v.so + j * v.sn + i * v.si);
        double out;
        if (KIND == 0) {
            const double mean = stats[c] / count;
            const double var = fmax(stats[cells + c] / count - mean * mean, 0.0);
            out = (xv - mean) / sqrt(var + eps);
        } else {
            using P = typename Pw<T>::type;
            out = (double)pw_exp((P)(xv - aux[c])) / stats[c];
        }
        y[o * vy.so + j * vy.sn + i * vy.si] = from_acc<T>(out);
    }
}

template <typename T>
__global__ void elementwise_k(int op, int64_t n, const T *__restrict__ a, const T *__restrict__ b,
                              double s, T *__restrict__ out) {
    using P = typename Pw<T>::type;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const P av = (P)ld64(a + e);
        const P bv = b ? (P)ld64(b + e) : (P)s;
        out[e] = from_acc<T>(op == 1 ? av * bv : (op == 0 ? av + bv : av * bv));
    }
}

int nsplit_for(const View3 &v) {
    const int64_t cells = v.outer * v.inner;
    const int64_t want = v.inner == 1 ? (int64_t)sm_count() * 32 : (int64_t)sm_count() * 1024;
    int64_t ns = cells >= want ? 1 : (want + cells - 1) / cells;
    const int64_t maxs = (v.n + 255) / 256;
    if (ns > maxs) ns = maxs;
    if (ns > 1024) ns = 1024;
    if (ns < 1) ns = 1;
    return (int)ns;
}

template <typename T>
int stats_t(int kind, const View3 &v, const void *x, const void *aux, void *stats, void *ws,
            cudaStream_t st) {
    const int ns = nsplit_for(v);
    const int64_t chunk = (v.n + ns - 1) / ns;
    const int64_t cells = v.outer * v.inner;
    const int64_t work = v.inner == 1 ? cells * ns * 32 : cells * ns;
    const int grid = grid_for(work, 256, 8);
    double *part = (double *)ws;
    const T *xp = (const T *)x;
    const double *ap = (const double *)aux;
    if (kind == 0)
        stats_partial<T, 0><<<grid, 256, 0, st>>>(v, xp, ap, part, chunk, ns);
    else if (kind == 1)
        stats_partial<T, 1><<<grid, 256, 0, st>>>(v, xp, ap, part, chunk, ns);
    else
        stats_partial<T, 2><<<grid, 256, 0, st>>>(v, xp, ap, part, chunk, ns);
    const int nstat = kind == 0 ? 2 : 1;
    stats_combine<<<grid_for(cells * nstat, 256, 4), 256, 0, st>>>(part, (double *)stats, cells,
                                                                   ns, nstat, kind == 1);
    return launch_status("dp_norm_stats", 2);
}

template <typename T>
int apply_t(int kind, const View3 &v, const void *x, void *y, const View3 &vy, const void *stats,
            const void *aux, double count, double eps, cudaStream_t st) {
    const int grid = grid_for(v.outer * v.n * v.inner, 256, 8);
    if (kind == 0)
        norm_apply<T, 0><<<grid, 256, 0, st>>>(v, (const T *)x, (T *)y, vy,
                                               (const double *)stats, (const double *)aux,
                                               count, eps);
    else
        norm_apply<T, 1><<<grid, 256, 0, st>>>(v, (const T *)x, (T *)y, vy,
                                               (const double *)stats, (const double *)aux,
                                               count, eps);
    return launch_status("dp_norm_apply");
}

bool view_ok(int64_t outer, int64_t n, int64_t inner, const int64_t *s) {
    return outer >= 0 && n >= 0 && inner >= 0 && s != nullptr;
}

}  // namespace
}  // namespace dp

using namespace dp;

extern "C" int64_t dp_norm_workspace(int kind, int64_t outer, int64_t n, int64_t inner) {
    View3 v{outer, n, inner, 0, 0, 0};
    if (outer < 0 || n < 0 || inner < 0 || kind < 0 || kind > 2) return -1;
    return (int64_t)nsplit_for(v) * outer * inner * (kind == 0 ? 2 : 1) * 8;
}

extern "C" int dp_norm_stats(int kind, int64_t outer, int64_t n, int64_t inner, const void *x,
                             const int64_t *xs, int dtype, const void *aux, void *stats, void *ws,
                             int64_t ws_bytes, void *stream) {
    DP_REQUIRE(view_ok(outer, n, inner, xs), DP_ERR_INVALID, "dp_norm_stats: bad view");
    DP_REQUIRE(kind >= 0 && kind <= 2, DP_ERR_INVALID, "dp_norm_stats: kind %d", kind);
    DP_REQUIRE(kind != 2 || aux, DP_ERR_INVALID, "dp_norm_stats: exp-sum needs the max");
    DP_REQUIRE(ws_bytes >= dp_norm_workspace(kind, outer, n, inner), DP_ERR_INVALID,
               "dp_norm_stats: workspace too small");
    if (outer * inner == 0) return DP_OK;
    View3 v{outer, n, inner, xs[0], xs[1], xs[2]};
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case DP_F32: return stats_t<float>(kind, v, x, aux, stats, ws, st);
        case DP_F64: return stats_t<double>(kind, v, x, aux, stats, ws, st);
        case DP_BF16: return stats_t<__nv_bfloat16>(kind, v, x, aux, stats, ws, st);
    }
    set_error("dp_norm_stats: dtype %d", dtype);
    return DP_ERR_UNSUPPORTED;
}

extern "C" int dp_norm_apply(int kind, int64_t outer, int64_t n, int64_t inner, const void *x,
                             const int64_t *xs, void *y, const int64_t *ys, int dtype,
                             const void *stats, const void *aux, double count, double eps,
                             void *stream) {
    DP_REQUIRE(view_ok(outer, n, inner, xs) && ys, DP_ERR_INVALID, "dp_norm_apply: bad view");
    DP_REQUIRE(kind == 0 || kind == 1, DP_ERR_INVALID, "dp_norm_apply: kind %d", kind);
    DP_REQUIRE(kind == 0 || aux, DP_ERR_INVALID, "dp_norm_apply: softmax needs the max");
    if (outer * n * inner == 0) return DP_OK;
    View3 v{outer, n, inner, xs[0], xs[1], xs[2]};
    View3 vy{outer, n, inner, ys[0], ys[1], ys[2]};
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case DP_F32: return apply_t<float>(kind, v, x, y, vy, stats, aux, count, eps, st);
        case DP_F64: return apply_t<double>(kind, v, x, y, vy, stats, aux, count, eps, st);
        case DP_BF16:
            return apply_t<__nv_bfloat16>(kind, v, x, y, vy, stats, aux, count, eps, st);
    }
    set_error("dp_norm_apply: dtype %d", dtype);
    return DP_ERR_UNSUPPORTED;
}

extern "C" int dp_elementwise(int op, int64_t n, const void *a, const void *b, double scalar,
                              void *out, int dtype, void *stream) {
    DP_REQUIRE(op >= 0 && op <= 2, DP_ERR_INVALID, "dp_elementwise: op %d", op);
    DP_REQUIRE(n >= 0 && (n == 0 || (a && out)), DP_ERR_INVALID, "dp_elementwise: bad args");
    if (n == 0) return DP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = grid_for(n, 256, 8);
    const void *bb = op == 2 ? nullptr : b;
    switch (dtype) {
        case DP_F32:
            elementwise_k<float><<<grid, 256, 0, st>>>(op, n, (const float *)a, (const float *)bb,
                                                       scalar, (float *)out);
            break;
        case DP_F64:
            elementwise_k<double><<<grid, 256, 0, st>>>(op, n, (const double *)a,
                                                        (const double *)bb, scalar,
                                                        (double *)out);
            break;
        case DP_BF16:
            elementwise_k<__nv_bfloat16><<<grid, 256, 0, st>>>(
                op, n, (const __nv_bfloat16 *)a, (const __nv_bfloat16 *)bb, scalar,
                (__nv_bfloat16 *)out);
            break;
        default:
            set_error("dp_elementwise: dtype %d", dtype);
            return DP_ERR_UNSUPPORTED;
    }
    return launch_status("dp_elementwise");
}
