// MUFU ex2 throughput probe: ops per clock per SM and ops/s chip-wide, the
// denominator of the attention forward's exp2 roofline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/mufu_probe scripts/mufu_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ex2_loop(float *out, int iters, long long *cyc) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    long long *cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 8);
    const int threads = 512, per_sm = 4, iters = 20000;
    const int blocks = sms * per_sm;
    ex2_loop<<<blocks, threads>>>(out, 100, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        ex2_loop<<<blocks, threads>>>(out, iters, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double ops = (double)blocks * threads * iters * 8;
        const double per_clk_sm = ops / sms / (double)c;   // block 0's clock span ~ the kernel
        printf("ex2.approx: %.3f Tops/s, %.2f ops/clk/SM (clock span %lld cyc, %.3f ms, %.0f MHz eff)\n",
               ops / (ms * 1e-3) / 1e12, per_clk_sm, c, ms, c / (ms * 1e3));
    }
    return 0;
}
