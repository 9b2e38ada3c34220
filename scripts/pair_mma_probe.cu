// Issue / execution rate of cta_group::2 tcgen05.mma (M = 256 over a CTA
// pair) vs cta_group::1 (M = 128) for the conv kernels' N = 48 / 96 shapes:
// NMMA back-to-back MMAs from one elected lane, one commit at the end,
// cycles per MMA.  SW64 K-major operands (the C_in = 32 conv layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_11111_b200/csrc \
//        -o scripts/bin/pair_mma_probe scripts/pair_mma_probe.cu -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace dp::tc;

template <bool PAIR, int N, int NACC = 1>
__global__ void __cluster_dims__(2, 1, 1) probe(int nmma, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x * 16; i < 64 * 1024; i += blockDim.x * 16)
        *reinterpret_cast<int4 *>(smem + i) = make_int4(0x3c003c00, 0x3c003c00, 0x3c003c00, 0x3c003c00);
    fence_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) {
        if (PAIR) tmem_alloc2(&tslot, 512);
        else tmem_alloc(&tslot, 512);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x < 32 && (!PAIR || rank == 0)) {
        const uint32_t id = idesc_bf16(PAIR ? 256 : 128, N);
        const uint64_t a0 = sdesc_sw(smem_u32(smem), 512, 4);            // SW64, 8 rows x 64 B
        const uint64_t b0 = sdesc_sw(smem_u32(smem + 32768), 512, 4);
        long long t0 = clock64();
        for (int i = 0; i < nmma; i += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t dacc = tmem + (uint32_t)((k % NACC) * N);   // NACC independent accumulators
                if (PAIR) mma2_bf16_e(dacc, a0 + (k & 1) * 2, b0 + (k & 1) * 2, id, 1u);
                else mma_bf16_e(dacc, a0 + (k & 1) * 2, b0 + (k & 1) * 2, id, 1u);
            }
        }
        if (PAIR) mma2_commit_mc_e(&bar);
        else mma_commit_e(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
    } else if (PAIR && threadIdx.x < 32) {
        mbar_wait(&bar, 0);   // the multicast commit arrives here too
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (threadIdx.x < 32) {
        if (PAIR) tmem_dealloc2(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

// the conv pair kernel's per-stage MMA-warp stream: 3 groups of 3 MMAs (x3),
// commits to two barriers (stage empty + row full), NSTAGE stages
template <int NG, int SW = 64, bool FENCE = false>
__global__ void __cluster_dims__(2, 1, 1) stage_probe(int nst, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bars[34];
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x * 16; i < 64 * 1024; i += blockDim.x * 16)
        *reinterpret_cast<int4 *>(smem + i) = make_int4(0x3c003c00, 0x3c003c00, 0x3c003c00, 0x3c003c00);
    fence_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 32; ++i) mbar_init(&bars[i], 1 << 20);
        mbar_init(&bars[32], 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc2(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x < 32 && rank == 0) {
        const uint32_t id = idesc_bf16(256, 96);
        // SW64: 8 rows x 64 B (C_in 32 layout); SW32: 8 rows x 32 B (C_in 16)
        const uint64_t a0 = sdesc_sw(smem_u32(smem), SW == 64 ? 512 : 256, SW == 64 ? 4 : 6);   // SW0: A SW32
        const uint64_t b0 = SW == 0 ? sdesc(smem_u32(smem + 32768), 128, 256)   // no-swizzle weight image
                                    : sdesc_sw(smem_u32(smem + 32768), SW == 64 ? 512 : 256, SW == 64 ? 4 : 6);
        long long t0 = clock64();
        for (int st = 0; st < nst; ++st) {
            if (FENCE) tc_fence_after();
            const uint32_t d = tmem + (st % 5) * 96;
#pragma unroll
            for (int g = 0; g < NG; ++g) mma2_bf16_x3<4, 96>(d, a0 + g * 64, b0 + g * 288, id);
            mma2_commit_mc_e(&bars[st & 15]);
            mma2_commit_mc_e(&bars[16 + (st & 15)]);
        }
        mma2_commit_mc_e(&bars[32]);
        mbar_wait(&bars[32], 0);
        long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (threadIdx.x < 32 && rank == 1) mbar_wait(&bars[32], 0);
    if (threadIdx.x < 32) tmem_dealloc2(tmem, 512);
}

template <int NG, int SW = 64, bool FENCE = false>
void run_stage(const char *name, long long *d) {
    const int nst = 2000;
    cudaFuncSetAttribute(stage_probe<NG, SW, FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int r = 0; r < 2; ++r) {
        stage_probe<NG, SW, FENCE><<<296, 128, 64 * 1024>>>(nst, d);
        cudaDeviceSynchronize();
    }
    long long h[296];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    int n = 0;
    for (int i = 0; i < 296; i += 2) { s += h[i]; ++n; }
    printf("%-34s %6.1f cycles / stage (%d MMAs)\n", name, s / n / nst, 3 * NG);
}

template <bool PAIR, int N, int NACC = 1>
void run(const char *name, long long *d) {
    const int nmma = 4096;
    cudaFuncSetAttribute(probe<PAIR, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int r = 0; r < 2; ++r) {
        probe<PAIR, N, NACC><<<296, 128, 64 * 1024>>>(nmma, d);
        cudaDeviceSynchronize();
    }
    long long h[296];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    int n = 0;
    for (int i = 0; i < 296; i += (PAIR ? 2 : 1)) { s += h[i]; ++n; }
    printf("%-34s %6.1f cycles / MMA\n", name, s / n / nmma);
}

int main() {
    long long *d;
    cudaMalloc(&d, 296 * sizeof(long long));
    run<false, 48>("cta_group::1 M=128 N=48", d);
    run<false, 96>("cta_group::1 M=128 N=96", d);
    run<false, 192>("cta_group::1 M=128 N=192", d);
    run<true, 48>("cta_group::2 M=256 N=48", d);
    run<true, 96>("cta_group::2 M=256 N=96", d);
    run<true, 192>("cta_group::2 M=256 N=192", d);
    run<false, 96, 2>("cta_group::1 N=96, 2 accumulators", d);
    run<true, 48, 2>("cta_group::2 N=48, 2 accumulators", d);
    run<true, 96, 2>("cta_group::2 N=96, 2 accumulators", d);
    run<true, 96, 4>("cta_group::2 N=96, 4 accumulators", d);
    run_stage<3>("stage: 3 x3 groups + 2 mc commits", d);
    run_stage<6>("stage: 6 x3 groups + 2 mc commits", d);
    run_stage<3, 32>("stage SW32: 3 x3 groups + 2 commits", d);
    run_stage<3, 0>("stage A SW32, B no-swizzle", d);
    run_stage<6, 0>("stage A SW32, B no-swizzle, 18", d);
    run_stage<3, 0, true>("stage 9 + tcgen05 fence per stage", d);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
