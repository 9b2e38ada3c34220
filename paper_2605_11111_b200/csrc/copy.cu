// Strided copy / accumulate / convert kernels: halo face pack/unpack, varlen
// redistribute pack/unpack, reverse-halo gradient accumulate, the
// accumulator -> parameter-dtype casts and fills of the ring backward, and
// the thread mesh's all_reduce fold.
//
// HBM-bound byte movement.  The host side collapses the index space
// (merging dims that are contiguous in BOTH src and dst), then moves the
// innermost run with the widest vector (16 B) both pointers and the run
// length allow.  The grid is a multiple of the SM count with a grid-stride
// loop; each thread keeps 4 independent vectors in flight.
#include <stdarg.h>

#include "common.cuh"

namespace dp {

static thread_local char g_err[1024];

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
const char *last_error() { return g_err; }

static unsigned long long g_launches = 0;
void note_launches(int n) { __atomic_add_fetch(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

int sm_count() {
    static int cached = 0;
    if (cached == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

namespace {

constexpr int kMaxDims = 8;

struct Walk {
    int nd;                 // number of outer dims (innermost run excluded)
    int64_t shape[kMaxDims];
    int64_t ss[kMaxDims];   // src strides, in units of the vector type
    int64_t ds[kMaxDims];   // dst strides, in units of the vector type
};

__device__ __forceinline__ void offsets(const Walk &w, int64_t row, int64_t &so, int64_t &d_o) {
    so = 0;
    d_o = 0;
#pragma unroll
    for (int i = kMaxDims - 1; i >= 0; --i) {
        if (i < w.nd) {
            int64_t n = w.shape[i];
            int64_t c = row % n;
            row /= n;
            so += c * w.ss[i];
            d_o += c * w.ds[i];
        }
    }
}

// Row-tiled walk: the index space is rows (outer dims) x `inner` vectors.
// G lanes (a power of two <= 32, ~ the row length) share a row: the row's
// source / destination offsets are computed once per row (64-bit div/mod
// amortised over the run) and the lanes stride over its vectors, 4
// independent loads in flight each.  Short rows (a 2-voxel halo face is 8
// x 16 B) pack 32/G rows per warp so no lane idles.
template <typename V, int G>
__global__ void __launch_bounds__(256) copy_rows(Walk w, int64_t inner, int64_t rows,
                                                 const V *__restrict__ src, V *__restrict__ dst) {
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    const int sub = threadIdx.x % G;
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; row < rows;
         row += groups) {
        int64_t so, d_o;
        offsets(w, row, so, d_o);
        const V *s = src + so;
        V *d = dst + d_o;
        int64_t c = sub;
        for (; c + 3 * G < inner; c += 4 * G) {
            V a0 = s[c], a1 = s[c + G], a2 = s[c + 2 * G], a3 = s[c + 3 * G];
            d[c] = a0;
            d[c + G] = a1;
            d[c + 2 * G] = a2;
            d[c + 3 * G] = a3;
        }
        for (; c < inner; c += G) d[c] = s[c];
    }
}

template <typename T>
__device__ __forceinline__ void acc_vec(T *d, const T *s);
template <>
__device__ __forceinline__ void acc_vec<float>(float *d, const float *s) {
    float4 a = *reinterpret_cast<const float4 *>(s);
    float4 b = *reinterpret_cast<float4 *>(d);
    b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
    *reinterpret_cast<float4 *>(d) = b;
}
template <>
__device__ __forceinline__ void acc_vec<double>(double *d, const double *s) {
    double2 a = *reinterpret_cast<const double2 *>(s);
    double2 b = *reinterpret_cast<double2 *>(d);
    b.x += a.x; b.y += a.y;
    *reinterpret_cast<double2 *>(d) = b;
}
template <>
__device__ __forceinline__ void acc_vec<__nv_bfloat16>(__nv_bfloat16 *d, const __nv_bfloat16 *s) {
    uint4 a = *reinterpret_cast<const uint4 *>(s);
    uint4 b = *reinterpret_cast<uint4 *>(d);
    __nv_bfloat162 *pa = reinterpret_cast<__nv_bfloat162 *>(&a);
    __nv_bfloat162 *pb = reinterpret_cast<__nv_bfloat162 *>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 x = __bfloat1622float2(pa[i]), y = __bfloat1622float2(pb[i]);
        pb[i] = __floats2bfloat162_rn(x.x + y.x, x.y + y.y);
    }
    *reinterpret_cast<uint4 *>(d) = b;
}
template <typename T> struct VecN { static constexpr int n = 16 / sizeof(T); };

// dst += src, row-tiled like copy_rows; VEC: 16-B vectors along a unit-stride
// inner run (fp32 adds in fp32, bf16 through fp32, fp64 in fp64).
template <typename T, int G, bool VEC>
__global__ void __launch_bounds__(256) accum_rows(Walk w, int64_t inner, int64_t rows,
                                                  int64_t s_inner, int64_t d_inner,
                                                  const T *__restrict__ src, T *__restrict__ dst) {
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    const int sub = threadIdx.x % G;
    constexpr int NV = VecN<T>::n;
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; row < rows;
         row += groups) {
        int64_t so, d_o;
        offsets(w, row, so, d_o);
        if (VEC) {
            for (int64_t c = sub; c < inner / NV; c += G)
                acc_vec<T>(dst + d_o + c * NV, src + so + c * NV);
        } else {
            for (int64_t c = sub; c < inner; c += G) {
                T *p = dst + d_o + c * d_inner;
                *p = from_acc<T>(to_acc(*p) + to_acc(src[so + c * s_inner]));
            }
        }
    }
}

int lanes_for(int64_t inner) {
    int g = 1;
    while (g < 32 && g < inner) g <<= 1;
    return g;
}

// Collapse (shape, src strides, dst strides) in place; returns new ndim.
// Dims of extent 1 are dropped; the rest are put in the destination's memory
// order (decreasing dst stride, ties by src stride) — every op here is an
// elementwise map, so the walk order is free, and a channels-last tensor
// (C innermost in memory, second in logical order) becomes one unit-stride
// run instead of an element-by-element walk; then neighbour dims merge when
// both tensors are contiguous across them.
int collapse(int nd, int64_t *shape, int64_t *ss, int64_t *ds) {
    int64_t sh[kMaxDims], a[kMaxDims], b[kMaxDims];
    int n = 0;
    for (int i = 0; i < nd; ++i) {
        if (shape[i] == 1) continue;
        sh[n] = shape[i];
        a[n] = ss[i];
        b[n] = ds[i];
        ++n;
    }
    for (int i = 1; i < n; ++i) {   // stable insertion sort, outermost first
        int64_t s0 = sh[i], a0 = a[i], b0 = b[i];
        int j = i - 1;
        while (j >= 0 && (b[j] < b0 || (b[j] == b0 && a[j] < a0))) {
            sh[j + 1] = sh[j];
            a[j + 1] = a[j];
            b[j + 1] = b[j];
            --j;
        }
        sh[j + 1] = s0;
        a[j + 1] = a0;
        b[j + 1] = b0;
    }
    if (n == 0) {
        shape[0] = 1;
        ss[0] = ds[0] = 1;
        return 1;
    }
    int m = 0;
    for (int i = 1; i < n; ++i) {
        if (a[m] == a[i] * sh[i] && b[m] == b[i] * sh[i]) {
            sh[m] *= sh[i];
            a[m] = a[i];
            b[m] = b[i];
        } else {
            ++m;
            sh[m] = sh[i];
            a[m] = a[i];
            b[m] = b[i];
        }
    }
    n = m + 1;
    for (int i = 0; i < n; ++i) {
        shape[i] = sh[i];
        ss[i] = a[i];
        ds[i] = b[i];
    }
    return n;
}

template <typename V, int G>
void launch_rows(const Walk &w, int64_t inner, int64_t rows, const void *src, void *dst,
                 cudaStream_t st) {
    const int64_t work = rows * ((inner + 4 * G - 1) / (4 * G)) * G;  // threads with work
    const int grid = grid_for((work + 0) / 1, 256, 16);
    copy_rows<V, G><<<grid, 256, 0, st>>>(w, inner, rows, (const V *)src, (V *)dst);
}

template <typename V>
int launch_copy(int n, const int64_t *shape, const int64_t *ss, const int64_t *ds, int vec_elems,
                const void *src, void *dst, cudaStream_t st) {
    Walk w;
    w.nd = n - 1;
    for (int i = 0; i < n - 1; ++i) {
        w.shape[i] = shape[i];
        w.ss[i] = ss[i] / vec_elems;
        w.ds[i] = ds[i] / vec_elems;
    }
    int64_t inner = shape[n - 1] / vec_elems;
    int64_t rows = 1;
    for (int i = 0; i < n - 1; ++i) rows *= shape[i];
    // long runs are cut into kChunk-vector rows (a new innermost outer dim)
    // so every SM gets rows; the tail of a run that does not divide goes in
    // a second launch
    constexpr int64_t kChunk = 2048;
    if (inner > 2 * kChunk && w.nd < kMaxDims) {
        const int64_t nch = inner / kChunk, rem = inner - nch * kChunk;
        if (rem) {
            Walk t = w;
            int64_t rrows = rows;
            const V *s2 = (const V *)src + nch * kChunk;
            V *d2 = (V *)dst + nch * kChunk;
            launch_rows<V, 32>(t, rem, rrows, s2, d2, st);
        }
        w.shape[w.nd] = nch;
        w.ss[w.nd] = kChunk;
        w.ds[w.nd] = kChunk;
        ++w.nd;
        rows *= nch;
        inner = kChunk;
    }
    switch (lanes_for(inner)) {
        case 1: launch_rows<V, 1>(w, inner, rows, src, dst, st); break;
        case 2: launch_rows<V, 2>(w, inner, rows, src, dst, st); break;
        case 4: launch_rows<V, 4>(w, inner, rows, src, dst, st); break;
        case 8: launch_rows<V, 8>(w, inner, rows, src, dst, st); break;
        case 16: launch_rows<V, 16>(w, inner, rows, src, dst, st); break;
        default: launch_rows<V, 32>(w, inner, rows, src, dst, st); break;
    }
    return launch_status("dp_copy_strided");
}

template <typename T, bool VEC>
int launch_accum(const Walk &w, int64_t inner, int64_t rows, int64_t s_in, int64_t d_in,
                 const void *src, void *dst, cudaStream_t st) {
    const int64_t units = VEC ? inner / VecN<T>::n : inner;
    const int g = lanes_for(units);
    const int grid = grid_for(rows * g, 256, 16);
#define DP_ACC(G)                                                                            \
    accum_rows<T, G, VEC><<<grid, 256, 0, st>>>(w, inner, rows, s_in, d_in, (const T *)src, \
                                                (T *)dst)
    switch (g) {
        case 1: DP_ACC(1); break;
        case 2: DP_ACC(2); break;
        case 4: DP_ACC(4); break;
        case 8: DP_ACC(8); break;
        case 16: DP_ACC(16); break;
        default: DP_ACC(32); break;
    }
#undef DP_ACC
    return launch_status("dp_accumulate_strided");
}

// ---------------------------------------------------------------------------
// typed element maps: converted copy (dst = (Td) src) and max-combine
// (dst = max(dst, src)); 4 elements per thread-step with vector loads /
// stores when the inner run is unit-stride and aligned (fp32 -> bf16 reads a
// float4 and writes 8 B), row-tiled like copy_rows.

template <typename T> struct V4;
template <> struct V4<float> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[4]) {
        float4 a = *reinterpret_cast<const float4 *>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
    static __device__ __forceinline__ void st(float *p, const float (&v)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <> struct V4<double> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[4]) {
        double2 a = reinterpret_cast<const double2 *>(p)[0], b = reinterpret_cast<const double2 *>(p)[1];
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    static __device__ __forceinline__ void st(double *p, const double (&v)[4]) {
        reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
    }
};
template <> struct V4<__nv_bfloat16> {
    static __device__ __forceinline__ void ld(const __nv_bfloat16 *p, __nv_bfloat16 (&v)[4]) {
        uint2 a = *reinterpret_cast<const uint2 *>(p);
        const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&a);
        v[0] = h[0]; v[1] = h[1]; v[2] = h[2]; v[3] = h[3];
    }
    static __device__ __forceinline__ void st(__nv_bfloat16 *p, const __nv_bfloat16 (&v)[4]) {
        uint2 a;
        __nv_bfloat16 *h = reinterpret_cast<__nv_bfloat16 *>(&a);
        h[0] = v[0]; h[1] = v[1]; h[2] = v[2]; h[3] = v[3];
        *reinterpret_cast<uint2 *>(p) = a;
    }
};

template <typename Td, typename Ts>
__device__ __forceinline__ Td cvt(Ts v) { return from_acc<Td>(to_acc(v)); }
template <> __device__ __forceinline__ double cvt<double, float>(float v) { return (double)v; }
template <> __device__ __forceinline__ float cvt<float, double>(double v) { return (float)v; }

template <typename Td, typename Ts, int OP>
__device__ __forceinline__ Td apply_op(Td d, Ts s) {
    if (OP == 0) return cvt<Td, Ts>(s);
    Td c = cvt<Td, Ts>(s);
    return to_acc(c) > to_acc(d) ? c : d;   // max; NaN in d stays, as max(nan, x)
}

// OP 0: dst = convert(src); OP 1: dst = max(dst, src)
template <typename Td, typename Ts, int OP, int G, bool VEC>
__global__ void __launch_bounds__(256) map_rows(Walk w, int64_t inner, int64_t rows,
                                                int64_t s_inner, int64_t d_inner,
                                                const Ts *__restrict__ src, Td *__restrict__ dst) {
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    const int sub = threadIdx.x % G;
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; row < rows;
         row += groups) {
        int64_t so, d_o;
        offsets(w, row, so, d_o);
        if (VEC) {
            for (int64_t c = sub; c < inner / 4; c += G) {
                Ts a[4];
                Td b[4];
                V4<Ts>::ld(src + so + 4 * c, a);
                if (OP == 1) V4<Td>::ld(dst + d_o + 4 * c, b);
#pragma unroll
                for (int k = 0; k < 4; ++k) b[k] = apply_op<Td, Ts, OP>(b[k], a[k]);
                V4<Td>::st(dst + d_o + 4 * c, b);
            }
        } else {
            for (int64_t c = sub; c < inner; c += G) {
                Td *p = dst + d_o + c * d_inner;
                *p = apply_op<Td, Ts, OP>(OP == 1 ? *p : Td(0), src[so + c * s_inner]);
            }
        }
    }
}

template <typename Td, typename Ts, int OP>
int launch_map(const Walk &w, int64_t inner, int64_t rows, int64_t s_in, int64_t d_in, bool vec,
               const void *src, void *dst, cudaStream_t st) {
    const int64_t units = vec ? inner / 4 : inner;
    const int g = lanes_for(units);
    const int grid = grid_for(rows * g, 256, 16);
#define DP_MAP(G)                                                                              \
    (vec ? map_rows<Td, Ts, OP, G, true><<<grid, 256, 0, st>>>(w, inner, rows, s_in, d_in,     \
                                                               (const Ts *)src, (Td *)dst)     \
         : map_rows<Td, Ts, OP, G, false><<<grid, 256, 0, st>>>(w, inner, rows, s_in, d_in,    \
                                                                (const Ts *)src, (Td *)dst))
    switch (g) {
        case 1: DP_MAP(1); break;
        case 2: DP_MAP(2); break;
        case 4: DP_MAP(4); break;
        case 8: DP_MAP(8); break;
        case 16: DP_MAP(16); break;
        default: DP_MAP(32); break;
    }
#undef DP_MAP
    return launch_status(OP == 0 ? "dp_convert_strided" : "dp_max_strided");
}

int elem_bytes_of(int dtype) { return dtype == DP_F64 ? 8 : dtype == DP_F32 ? 4 : 2; }

template <int OP>
int map_strided(int ndim, const int64_t *shape, void *dst, const int64_t *dst_strides, int dt_d,
                const void *src, const int64_t *src_strides, int dt_s, cudaStream_t st) {
    DP_REQUIRE(ndim >= 1 && ndim <= 8, DP_ERR_INVALID, "element map: ndim %d out of [1,8]", ndim);
    DP_REQUIRE((dt_d == DP_F32 || dt_d == DP_F64 || dt_d == DP_BF16) &&
                   (dt_s == DP_F32 || dt_s == DP_F64 || dt_s == DP_BF16),
               DP_ERR_INVALID, "element map: dtypes %d <- %d", dt_d, dt_s);
    int64_t sh[8], ss[8], ds[8];
    int64_t total = 1;
    for (int i = 0; i < ndim; ++i) {
        DP_REQUIRE(shape[i] >= 0, DP_ERR_INVALID, "element map: negative extent");
        sh[i] = shape[i];
        ss[i] = src_strides[i];
        ds[i] = dst_strides[i];
        total *= shape[i];
    }
    if (total == 0) return DP_OK;
    DP_REQUIRE(src && dst, DP_ERR_INVALID, "element map: null pointer");
    int n = collapse(ndim, sh, ss, ds);
    Walk w;
    w.nd = n - 1;
    for (int i = 0; i < n - 1; ++i) {
        w.shape[i] = sh[i];
        w.ss[i] = ss[i];
        w.ds[i] = ds[i];
    }
    int64_t inner = sh[n - 1];
    int64_t rows = total / inner;
    const int eb_s = elem_bytes_of(dt_s), eb_d = elem_bytes_of(dt_d);
    if (inner > 16384 && ss[n - 1] == 1 && ds[n - 1] == 1 && w.nd < 8) {
        constexpr int64_t kChunk = 8192;
        const int64_t nch = inner / kChunk, rem = inner - nch * kChunk;
        if (rem) {
            int64_t tsh[8], tss[8], tds[8];
            for (int i = 0; i < n; ++i) {
                tsh[i] = sh[i];
                tss[i] = ss[i];
                tds[i] = ds[i];
            }
            tsh[n - 1] = rem;
            int rc = map_strided<OP>(n, tsh, (char *)dst + nch * kChunk * eb_d, tds, dt_d,
                                     (const char *)src + nch * kChunk * eb_s, tss, dt_s, st);
            if (rc) return rc;
        }
        w.shape[w.nd] = nch;
        w.ss[w.nd] = kChunk;
        w.ds[w.nd] = kChunk;
        ++w.nd;
        rows *= nch;
        inner = kChunk;
    }
    bool vec = ss[n - 1] == 1 && ds[n - 1] == 1 && inner % 4 == 0 &&
               (uintptr_t)src % (4 * eb_s) == 0 && (uintptr_t)dst % (4 * eb_d) == 0;
    for (int i = 0; i < w.nd && vec; ++i) vec = w.ss[i] % 4 == 0 && w.ds[i] % 4 == 0;
    const int64_t si = ss[n - 1], di = ds[n - 1];
#define DP_PAIR(TD, TS) return launch_map<TD, TS, OP>(w, inner, rows, si, di, vec, src, dst, st)
    switch (dt_d * 3 + dt_s) {
        case DP_F32 * 3 + DP_F32: DP_PAIR(float, float);
        case DP_F32 * 3 + DP_F64: DP_PAIR(float, double);
        case DP_F32 * 3 + DP_BF16: DP_PAIR(float, __nv_bfloat16);
        case DP_F64 * 3 + DP_F32: DP_PAIR(double, float);
        case DP_F64 * 3 + DP_F64: DP_PAIR(double, double);
        case DP_F64 * 3 + DP_BF16: DP_PAIR(double, __nv_bfloat16);
        case DP_BF16 * 3 + DP_F32: DP_PAIR(__nv_bfloat16, float);
        case DP_BF16 * 3 + DP_F64: DP_PAIR(__nv_bfloat16, double);
        default: DP_PAIR(__nv_bfloat16, __nv_bfloat16);
    }
#undef DP_PAIR
}

// fill: n elements of dtype with `value` (zero -> cudaMemsetAsync)
template <typename T>
__global__ void __launch_bounds__(256) fill_kernel(T *__restrict__ dst, int64_t n, T v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = v;
}

}  // namespace
}  // namespace dp

using namespace dp;

extern "C" int dp_abi_version(void) { return DP_ABI_VERSION; }
extern "C" const char *dp_last_error(void) { return dp::last_error(); }
extern "C" uint64_t dp_launch_count(void) {
    return __atomic_load_n(&dp::g_launches, __ATOMIC_RELAXED);
}

extern "C" int dp_device_info(int *sms, int *major, int *minor) {
    int dev = 0;
    DP_CUDA_CHECK(cudaGetDevice(&dev));
    if (sms) *sms = dp::sm_count();
    if (major) DP_CUDA_CHECK(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev));
    if (minor) DP_CUDA_CHECK(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev));
    return DP_OK;
}

extern "C" int dp_copy_strided(int ndim, const int64_t *shape, void *dst, const int64_t *dst_strides,
                               const void *src, const int64_t *src_strides, int elem_bytes,
                               void *stream) {
    DP_REQUIRE(ndim >= 1 && ndim <= 8, DP_ERR_INVALID, "dp_copy_strided: ndim %d out of [1,8]", ndim);
    DP_REQUIRE(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8 ||
                   elem_bytes == 16,
               DP_ERR_INVALID, "dp_copy_strided: elem_bytes %d", elem_bytes);
    int64_t sh[8], ss[8], ds[8];
    int64_t total = 1;
    for (int i = 0; i < ndim; ++i) {
        DP_REQUIRE(shape[i] >= 0, DP_ERR_INVALID, "dp_copy_strided: negative extent");
        sh[i] = shape[i];
        ss[i] = src_strides[i];
        ds[i] = dst_strides[i];
        total *= shape[i];
    }
    if (total == 0) return DP_OK;
    DP_REQUIRE(src && dst, DP_ERR_INVALID, "dp_copy_strided: null pointer");
    int n = collapse(ndim, sh, ss, ds);
    // widen the element when the innermost run is unit-stride in both
    int64_t run_bytes = (ss[n - 1] == 1 && ds[n - 1] == 1) ? sh[n - 1] * elem_bytes : elem_bytes;
    int vec_bytes = elem_bytes;
    if (ss[n - 1] == 1 && ds[n - 1] == 1) {
        for (int vb = 16; vb > elem_bytes; vb >>= 1) {
            bool ok = (run_bytes % vb == 0) && ((uintptr_t)src % vb == 0) &&
                      ((uintptr_t)dst % vb == 0);
            for (int i = 0; i < n - 1 && ok; ++i)
                ok = ((ss[i] * elem_bytes) % vb == 0) && ((ds[i] * elem_bytes) % vb == 0);
            if (ok) {
                vec_bytes = vb;
                break;
            }
        }
    } else {
        // innermost dim is strided: append a unit inner dim so the walker
        // handles it as an outer dim
        DP_REQUIRE(n < 8, DP_ERR_UNSUPPORTED, "dp_copy_strided: too many strided dims");
        sh[n] = 1;
        ss[n] = 1;
        ds[n] = 1;
        ++n;
    }
    int ve = vec_bytes / elem_bytes;
    // strides are in elements; convert to vector units inside launch_copy
    int64_t shv[8];
    for (int i = 0; i < n; ++i) shv[i] = sh[i];
    cudaStream_t st = (cudaStream_t)stream;
    switch (vec_bytes) {
        case 16: return launch_copy<int4>(n, shv, ss, ds, ve, src, dst, st);
        case 8: return launch_copy<int2>(n, shv, ss, ds, ve, src, dst, st);
        case 4: return launch_copy<int>(n, shv, ss, ds, ve, src, dst, st);
        case 2: return launch_copy<short>(n, shv, ss, ds, ve, src, dst, st);
        default: return launch_copy<char>(n, shv, ss, ds, ve, src, dst, st);
    }
}

extern "C" int dp_accumulate_strided(int ndim, const int64_t *shape, void *dst,
                                     const int64_t *dst_strides, const void *src,
                                     const int64_t *src_strides, int dtype, void *stream) {
    DP_REQUIRE(ndim >= 1 && ndim <= 8, DP_ERR_INVALID, "dp_accumulate_strided: ndim %d", ndim);
    int64_t sh[8], ss[8], ds[8];
    int64_t total = 1;
    for (int i = 0; i < ndim; ++i) {
        sh[i] = shape[i];
        ss[i] = src_strides[i];
        ds[i] = dst_strides[i];
        total *= shape[i];
    }
    if (total == 0) return DP_OK;
    int n = collapse(ndim, sh, ss, ds);
    Walk w;
    w.nd = n - 1;
    for (int i = 0; i < n - 1; ++i) {
        w.shape[i] = sh[i];
        w.ss[i] = ss[i];
        w.ds[i] = ds[i];
    }
    int64_t inner = sh[n - 1];
    int64_t rows = total / inner;
    cudaStream_t st = (cudaStream_t)stream;
    const int eb = dtype == DP_F64 ? 8 : dtype == DP_F32 ? 4 : 2;
    // long unit-stride runs: cut into 8192-element rows (tail in a 2nd launch)
    if (inner > 16384 && ss[n - 1] == 1 && ds[n - 1] == 1 && w.nd < 8) {
        constexpr int64_t kChunk = 8192;
        const int64_t nch = inner / kChunk, rem = inner - nch * kChunk;
        if (rem) {
            int64_t tsh[8], tss[8], tds[8];
            for (int i = 0; i < n; ++i) {
                tsh[i] = sh[i];
                tss[i] = ss[i];
                tds[i] = ds[i];
            }
            tsh[n - 1] = rem;
            const char *s2 = (const char *)src + nch * kChunk * eb;
            char *d2 = (char *)dst + nch * kChunk * eb;
            int rc = dp_accumulate_strided(n, tsh, d2, tds, s2, tss, dtype, stream);
            if (rc) return rc;
        }
        w.shape[w.nd] = nch;
        w.ss[w.nd] = kChunk;
        w.ds[w.nd] = kChunk;
        ++w.nd;
        rows *= nch;
        inner = kChunk;
    }
    // 16-B vectors when the inner run is unit-stride on both sides and every
    // row start is 16-B aligned
    bool vec = ss[n - 1] == 1 && ds[n - 1] == 1 && (inner * eb) % 16 == 0 &&
               (uintptr_t)src % 16 == 0 && (uintptr_t)dst % 16 == 0;
    for (int i = 0; i < n - 1 && vec; ++i)
        vec = (ss[i] * eb) % 16 == 0 && (ds[i] * eb) % 16 == 0;
    switch (dtype) {
        case DP_F32:
            return vec ? launch_accum<float, true>(w, inner, rows, ss[n - 1], ds[n - 1], src, dst, st)
                       : launch_accum<float, false>(w, inner, rows, ss[n - 1], ds[n - 1], src, dst, st);
        case DP_F64:
            return vec ? launch_accum<double, true>(w, inner, rows, ss[n - 1], ds[n - 1], src, dst, st)
                       : launch_accum<double, false>(w, inner, rows, ss[n - 1], ds[n - 1], src, dst, st);
        case DP_BF16:
            return vec ? launch_accum<__nv_bfloat16, true>(w, inner, rows, ss[n - 1], ds[n - 1], src,
                                                           dst, st)
                       : launch_accum<__nv_bfloat16, false>(w, inner, rows, ss[n - 1], ds[n - 1],
                                                            src, dst, st);
        default:
            set_error("dp_accumulate_strided: dtype %d", dtype);
            return DP_ERR_INVALID;
    }
}

extern "C" int dp_convert_strided(int ndim, const int64_t *shape, void *dst,
                                  const int64_t *dst_strides, int dst_dtype, const void *src,
                                  const int64_t *src_strides, int src_dtype, void *stream) {
    return map_strided<0>(ndim, shape, dst, dst_strides, dst_dtype, src, src_strides, src_dtype,
                          (cudaStream_t)stream);
}

extern "C" int dp_max_strided(int ndim, const int64_t *shape, void *dst, const int64_t *dst_strides,
                              const void *src, const int64_t *src_strides, int dtype,
                              void *stream) {
    return map_strided<1>(ndim, shape, dst, dst_strides, dtype, src, src_strides, dtype,
                          (cudaStream_t)stream);
}

extern "C" int dp_fill(int64_t n, void *dst, int dtype, double value, void *stream) {
    DP_REQUIRE(n >= 0, DP_ERR_INVALID, "dp_fill: negative count");
    DP_REQUIRE(dtype == DP_F32 || dtype == DP_F64 || dtype == DP_BF16, DP_ERR_INVALID,
               "dp_fill: dtype %d", dtype);
    if (n == 0) return DP_OK;
    DP_REQUIRE(dst, DP_ERR_INVALID, "dp_fill: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int eb = elem_bytes_of(dtype);
    if (value == 0.0 && !signbit(value)) {
        DP_CUDA_CHECK(cudaMemsetAsync(dst, 0, (size_t)n * eb, st));
        return DP_OK;
    }
    const int grid = grid_for(n, 256, 8);
    if (dtype == DP_F32)
        fill_kernel<float><<<grid, 256, 0, st>>>((float *)dst, n, (float)value);
    else if (dtype == DP_F64)
        fill_kernel<double><<<grid, 256, 0, st>>>((double *)dst, n, value);
    else
        fill_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((__nv_bfloat16 *)dst, n,
                                                         __float2bfloat16_rn((float)value));
    return launch_status("dp_fill");
}
