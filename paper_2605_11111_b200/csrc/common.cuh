// Shared helpers for the sm_100a kernels behind include/dp_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/dp_b200.h"

namespace dp {

// ---------------------------------------------------------------------------
// error reporting across the C ABI (thread-local last message)

void set_error(const char *fmt, ...);
const char *last_error();

#define DP_REQUIRE(cond, code, ...)           \
    do {                                      \
        if (!(cond)) {                        \
            ::dp::set_error(__VA_ARGS__);     \
            return (code);                    \
        }                                     \
    } while (0)

#define DP_CUDA_CHECK(expr)                                                             \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            ::dp::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                            __FILE__, __LINE__);                                        \
            return DP_ERR_CUDA;                                                         \
        }                                                                               \
    } while (0)

void note_launches(int n);

// Check the last launch(es) and count `n` kernel launches for dp_launch_count().
inline int launch_status(const char *what, int n = 1) {
    note_launches(n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s launch failed: %s", what, cudaGetErrorString(e));
        return DP_ERR_CUDA;
    }
    return DP_OK;
}

int sm_count();

// ---------------------------------------------------------------------------
// element types

template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_acc(float v) { return v; }
__device__ __forceinline__ double to_acc(double v) { return v; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_acc(float v) { return (T)v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}
template <typename T> __device__ __forceinline__ T from_acc(double v) { return (T)v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(double v) {
    return __float2bfloat16_rn((float)v);
}

__device__ __forceinline__ float acc_exp(float v) { return expf(v); }
__device__ __forceinline__ double acc_exp(double v) { return exp(v); }
__device__ __forceinline__ float acc_log(float v) { return logf(v); }
__device__ __forceinline__ double acc_log(double v) { return log(v); }

template <typename T> __device__ __forceinline__ T neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -INFINITY; }

inline int grid_for(int64_t work, int block, int waves_per_sm = 8) {
    int64_t g = (work + block - 1) / block;
    int64_t cap = (int64_t)sm_count() * waves_per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace dp
