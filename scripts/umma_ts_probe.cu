// Probe: tcgen05.mma kind::f16 with the A operand in TMEM ("TS" form).
// Checks the assumed layout (lane m = row m; 32-bit column c of a K=16 step
// holds elements k = 2c, 2c+1 as bf16x2) against a host reference, and
// times it.  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
constexpr int M = 128, N = 64, K = 64;

// A [M][K] bf16 row-major (global), B [N][K] bf16 row-major (global), D [M][N] fp32
__global__ void probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D, int iters, long long *cyc) {
    __shared__ __align__(1024) uint8_t bs[N * K * 2];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // B into smem, K-major SWIZZLE_NONE canonical: core matrix = 8 rows x 16 B;
    // [n/8][k/8][8 rows][8 k]  -> SBO (8-row groups) = (K/8)*128, LBO (k halves) = 128
    for (int e = tid; e < N * K; e += blockDim.x) {
        int n = e / K, k = e % K;
        int off = ((n / 8) * (K / 8) + (k / 8)) * 64 + (n % 8) * 8 + (k % 8);
        reinterpret_cast<__nv_bfloat16 *>(bs)[off] = B[n * K + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint32_t colA = 128, colD = 0;   // A: K/2 = 32 columns at 128; D: N = 64 columns at 0
    // A into TMEM: thread (warp w, lane) = row 32w + lane; column c = (A[2c], A[2c+1])
    {
        const int m = warp * 32 + lane;
        uint32_t r[16];
        for (int c0 = 0; c0 < K / 2; c0 += 16) {
            for (int i = 0; i < 16; ++i) {
                __nv_bfloat162 v;
                v.x = A[m * K + 2 * (c0 + i)];
                v.y = A[m * K + 2 * (c0 + i) + 1];
                r[i] = *reinterpret_cast<uint32_t *>(&v);
            }
            const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + colA + c0;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                :: "r"(addr), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) {
        const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t b0 = desc_none(smem_u32(bs), 128, (K / 8) * 128);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int ks = 0; ks < K / 16; ++ks) {
                const uint32_t a = tmem + colA + ks * 8;                   // 8 columns per K=16 step
                const uint64_t b = b0 + ((ks * 2 * 128) >> 4);            // two 8-k core matrices
                const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
                asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                             "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                             ::"r"(tmem + colD), "r"(a), "l"(b), "r"(id), "r"(acc));
            }
        }
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
        long long t1 = clock64();
        if (lane == 0) *cyc = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {
        const int m = warp * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t r[16];
            const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + colD + c0;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 16; ++i) D[m * N + c0 + i] = __uint_as_float(r[i]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
    __nv_bfloat16 *hA = new __nv_bfloat16[M * K], *hB = new __nv_bfloat16[N * K];
    float *fa = new float[M * K], *fb = new float[N * K];
    unsigned s = 1;
    for (int i = 0; i < M * K; ++i) { s = s * 1103515245 + 12345; fa[i] = ((s >> 16) % 17) / 8.0f - 1.0f; hA[i] = __float2bfloat16(fa[i]); fa[i] = __bfloat162float(hA[i]); }
    for (int i = 0; i < N * K; ++i) { s = s * 1103515245 + 12345; fb[i] = ((s >> 16) % 13) / 8.0f - 0.75f; hB[i] = __float2bfloat16(fb[i]); fb[i] = __bfloat162float(hB[i]); }
    __nv_bfloat16 *dA, *dB; float *dD; long long *dc;
    cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
    for (int iters : {1, 512}) {
        probe<<<1, 128>>>(dA, dB, dD, iters, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        float *hD = new float[M * N]; long long cyc;
        cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)fa[m * K + k] * fb[n * K + k];
                ref *= iters;
                maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]) / (fabs(ref) + 1));
            }
        printf("iters %d: max rel err %.3e ; %.1f cycles per M=128 N=%d K=16 TS mma\n", iters, maxerr,
               (double)cyc / (iters * (K / 16)), N);
    }
    return 0;
}
