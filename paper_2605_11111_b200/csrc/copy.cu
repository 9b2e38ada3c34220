// Strided copy / accumulate kernels: halo face pack/unpack, varlen
// redistribute pack/unpack, reverse-halo gradient accumulate.
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

template <typename V>
__global__ void __launch_bounds__(256) copy_kernel(Walk w, int64_t inner, int64_t total,
                                                   const V *__restrict__ src, V *__restrict__ dst) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // 4 vectors in flight per thread
    for (; i < total; i += 4 * stride) {
        V buf[4];
        int64_t dofs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int64_t j = i + u * stride;
            if (j < total) {
                int64_t row = j / inner, col = j - row * inner, so, d_o;
                offsets(w, row, so, d_o);
                buf[u] = src[so + col];
                dofs[u] = d_o + col;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int64_t j = i + u * stride;
            if (j < total) dst[dofs[u]] = buf[u];
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) accum_kernel(Walk w, int64_t inner, int64_t total,
                                                    int64_t s_inner, int64_t d_inner,
                                                    const T *__restrict__ src, T *__restrict__ dst) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride) {
        int64_t row = j / inner, col = j - row * inner, so, d_o;
        offsets(w, row, so, d_o);
        T *p = dst + d_o + col * d_inner;
        *p = from_acc<T>(to_acc(*p) + to_acc(src[so + col * s_inner]));
    }
}

// Collapse (shape, src strides, dst strides) in place; returns new ndim.
// Dims of extent 1 are dropped; neighbour dims merge when both tensors are
// contiguous across them.
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
    int64_t total = rows * inner;
    int grid = grid_for((total + 3) / 4, 256, 16);
    copy_kernel<V><<<grid, 256, 0, st>>>(w, inner, total, (const V *)src, (V *)dst);
    return launch_status("dp_copy_strided");
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
    int grid = grid_for(total, 256, 16);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case DP_F32:
            accum_kernel<float><<<grid, 256, 0, st>>>(w, inner, total, ss[n - 1], ds[n - 1],
                                                     (const float *)src, (float *)dst);
            break;
        case DP_F64:
            accum_kernel<double><<<grid, 256, 0, st>>>(w, inner, total, ss[n - 1], ds[n - 1],
                                                      (const double *)src, (double *)dst);
            break;
        case DP_BF16:
            accum_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
                w, inner, total, ss[n - 1], ds[n - 1], (const __nv_bfloat16 *)src,
                (__nv_bfloat16 *)dst);
            break;
        default:
            set_error("dp_accumulate_strided: dtype %d", dtype);
            return DP_ERR_INVALID;
    }
    return launch_status("dp_accumulate_strided");
}
