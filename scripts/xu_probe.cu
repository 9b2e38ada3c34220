// Issue/pipe throughput of the attention softmax instruction mix on one SM:
// MUFU.EX2 alone, F2FP (cvt.rn.bf16x2.f32) alone, and both interleaved —
// whether the bf16 packs share the MUFU (XU) pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/xu_probe scripts/xu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float *out, int iters) {
    float a[8];
    uint32_t acc = 0;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE & 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (MODE & 2) {
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                acc += r;
            }
            if (MODE & 4) {   // round-half-up pack via integer ops
                uint32_t x = __float_as_uint(a[i]) + 0x8000u, y = __float_as_uint(a[(i + 1) & 7]) + 0x8000u;
                uint32_t r;
                asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(x), "r"(y));
                acc += r;
            }
        }
    }
    long long t1 = clock64();
    float s = acc;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}
template <int M>
void run(const char *name, float *d) {
    const int iters = 4096;
    for (int r = 0; r < 2; ++r) { k<M><<<148, 512>>>(d, iters); cudaDeviceSynchronize(); }
    float c;
    cudaMemcpy(&c, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    // per SM: 16 warps x iters x 8 ops
    printf("%-28s %6.2f cycles per warp-op per SM (%.1f lanes/clk)\n", name, c / (16.0 * iters * 8),
           32.0 * 16 * iters * 8 / c);
}
int main() {
    float *d;
    cudaMalloc(&d, (1 << 20) * 4 + 64);
    run<1>("MUFU.EX2", d);
    run<2>("F2FP bf16x2 pack", d);
    run<3>("EX2 + F2FP", d);
    run<4>("IADD+PRMT pack", d);
    run<5>("EX2 + IADD/PRMT pack", d);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
