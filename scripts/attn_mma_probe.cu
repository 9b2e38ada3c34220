// Tensor-pipe throughput of the attention backward's per-block MMA stream
// (csrc/attn_tc.cu attn_bwd_tc_kernel), issued back to back without any
// synchronisation: S^T / dP^T (SS, K-major SW128, 4 or 5 K steps), dV (TS,
// B MN-major), dK (SS, A K-major, B MN-major), dQ (SS, A and B MN-major).
// One CTA per SM; cycles per block for each group alone and for the mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/attn_mma_probe scripts/attn_mma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void commit_to(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
template <int mode>
__global__ void probe(int nblk, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, cb[6];
    {
        uint32_t hsh = 0x9e3779b9u * (threadIdx.x + 1 + blockIdx.x * 977);
        for (int i = threadIdx.x * 4; i < 200 * 1024; i += blockDim.x * 4) {
            uint32_t v = 0;
            if (mode & 2048) {   // random bf16 pairs, |x| in [0.5, 2)
                hsh ^= hsh << 13; hsh ^= hsh >> 17; hsh ^= hsh << 5;
                v = ((hsh & 0x80008000u) | 0x3f003f00u) + ((hsh >> 4) & 0x00ff00ffu);
            } else {
                v = 0x3c003c00u;
            }
            *reinterpret_cast<uint32_t *>(smem + i) = v;
        }
    }
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        for (int i = 0; i < 6; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cb[i])), "r"(1 << 20));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp >= 4 && (mode & (64 | 128))) {
        // background load: 8 warps of TMEM reads (64) and / or LSU shared traffic (128)
        uint32_t acc = 0;
        const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint8_t *my = smem + 90112 + (threadIdx.x & 255) * 16;   // dS^T-like region
        while (!stop) {
            if constexpr (mode & 64) {
                uint32_t r[16];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                             : "r"(lb + ((warp >> 2) & 1) * 64));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                for (int i = 0; i < 16; ++i) acc += r[i];
            }
            if constexpr (mode & 128) {
                for (int i = 0; i < 8; ++i) {
                    int4 v;
                    asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(smem_u32(smem + 180224 + i * 16)));   // broadcast
                    acc += v.x;
                    asm volatile("st.shared.v4.s32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(my + (i & 1) * 4096)),
                                 "r"((int)acc), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
                }
            }
        }
        if (acc == 0x12345) out[200] = acc;
    }
    if (threadIdx.x == 0) {
        const uint32_t K = 0, V = 16384, Q = 32768, DO = 49152, AUG = 65536, DS = 73728;
        const uint32_t base = smem_u32(smem);
        const uint32_t id_s = idesc(128, 128, 0, 0), id_g = idesc(128, 64, 0, 1), id_q = idesc(128, 64, 1, 1);
        const uint64_t kd = sdesc(base + K, 16, 1024, 2), vd = sdesc(base + V, 16, 1024, 2);
        const uint64_t qk = sdesc(base + Q, 16, 1024, 2), dok = sdesc(base + DO, 16, 1024, 2);
        const uint64_t ka = sdesc(base + AUG, 16, 256, 6);
        const uint64_t q_mn = sdesc(base + Q, 8192, 1024, 2), do_mn = sdesc(base + DO, 8192, 1024, 2);
        const uint64_t kmn = sdesc(base + K, 8192, 1024, 2);
        const uint64_t dst_k = sdesc(base + DS, 16, 1024, 2), ds_mn = sdesc(base + DS, 16384, 1024, 2);
        long long t0 = clock64();
#pragma unroll 1
        for (int j = 0; j < nblk; ++j) {
            if constexpr (mode & 1) {
                for (int k = 0; k < 4; ++k) {
                    mma_ss(tmem + 0, kd + ((k * 32) >> 4), qk + ((k * 32) >> 4), id_s, k ? 1u : 0u);
                    mma_ss(tmem + 128, vd + ((k * 32) >> 4), dok + ((k * 32) >> 4), id_s, k ? 1u : 0u);
                }
                if constexpr (mode & 32) {
                    mma_ss(tmem + 0, ka, ka, id_s, 1u);
                    mma_ss(tmem + 128, ka, ka, id_s, 1u);
                }
                if constexpr (mode & 256) commit_to(&cb[0]);
            }
            if constexpr (mode & 2)
                for (int k = 0; k < 8; ++k)
                    mma_ts(tmem + 256, tmem + 448 + k * 8, do_mn + ((k * 16 * 128) >> 4), id_g, 1u);
            if constexpr ((mode & 256) && (mode & 2)) commit_to(&cb[1]);
            if constexpr (mode & 4)
                for (int k = 0; k < 8; ++k)
                    mma_ss(tmem + 320, dst_k + (((k >> 2) * (128 * 128) + (k & 3) * 32) >> 4),
                           q_mn + ((k * 16 * 128) >> 4), id_g, 1u);
            if constexpr (mode & 8)
                for (int k = 0; k < 8; ++k)
                    mma_ss(tmem + 384, ds_mn + ((k * 16 * 128) >> 4), kmn + ((k * 16 * 128) >> 4), id_q, k ? 1u : 0u);
            if constexpr (mode & 256) { commit_to(&cb[2]); commit_to(&cb[3]); commit_to(&cb[4]); }
            if constexpr (mode & 512)   // dV, dK, dQ k-steps interleaved (three accumulators in flight)
                for (int k = 0; k < 8; ++k) {
                    mma_ts(tmem + 256, tmem + 448 + k * 8, do_mn + ((k * 16 * 128) >> 4), id_g, 1u);
                    mma_ss(tmem + 320, dst_k + (((k >> 2) * (128 * 128) + (k & 3) * 32) >> 4),
                           q_mn + ((k * 16 * 128) >> 4), id_g, 1u);
                    mma_ss(tmem + 384, ds_mn + ((k * 16 * 128) >> 4), kmn + ((k * 16 * 128) >> 4), id_q, k ? 1u : 0u);
                }
            if constexpr (mode & 1024)   // dK, dQ interleaved after dV
                for (int k = 0; k < 8; ++k) {
                    mma_ss(tmem + 320, dst_k + (((k >> 2) * (128 * 128) + (k & 3) * 32) >> 4),
                           q_mn + ((k * 16 * 128) >> 4), id_g, 1u);
                    mma_ss(tmem + 384, ds_mn + ((k * 16 * 128) >> 4), kmn + ((k * 16 * 128) >> 4), id_q, k ? 1u : 0u);
                }
            if constexpr (mode & 16)   // dK as TS (A = dS^T from TMEM), for comparison
                for (int k = 0; k < 8; ++k)
                    mma_ts(tmem + 320, tmem + 448 + k * 8, q_mn + ((k * 16 * 128) >> 4), id_g, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        stop = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int M>
void run(const char *name, long long *d, int nblk) {
    cudaFuncSetAttribute(probe<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
        probe<M><<<148, 384, 200 * 1024>>>(nblk, d);
        cudaDeviceSynchronize();
    }
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    printf("%-26s %8.1f cycles/block\n", name, avg / 148 / nblk);
}

int main() {
    long long *d;
    cudaMalloc(&d, 256 * sizeof(long long));
    const int n = 2000;
    run<1>("S+dP (4 K steps)", d, n);
    run<33>("S+dP (5 K steps, aug)", d, n);
    run<2>("dV TS", d, n);
    run<4>("dK SS", d, n);
    run<16>("dK TS", d, n);
    run<8>("dQ SS mn/mn", d, n);
    run<15>("all (current)", d, n);
    run<15 | 64>("all + TMEM ld load", d, n);
    run<15 | 128>("all + LSU smem load", d, n);
    run<15 | 256>("all + 5 commits/block", d, n);
    run<512>("grads interleaved", d, n);
    run<2 | 4 | 8>("grads sequential", d, n);
    run<1 | 512>("S+dP, grads interleaved", d, n);
    run<1 | 2 | 1024>("S+dP, dV, dK||dQ", d, n);
    run<1 | 2 | 16 | 8>("S+dP, dV, dK TS, dQ", d, n);
    run<15 | 2048>("all, random data", d, n);
    run<1 | 2048>("S+dP, random data", d, n);
    run<15 | 2048 | 64 | 128 | 256>("all, random, loads, commits", d, n);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
