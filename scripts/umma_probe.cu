// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1, M=128)
// for several N and shared-memory operand layouts.  Not part of the
// library; used to pick the conv/attention operand layouts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn = 0, int b_mn = 0) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct Cfg { int dcol; int epi; int N; int alayout; uint32_t alab, asbo; int blayout; uint32_t blbo, bsbo; int ashift; int a_mn; int b_mn; };

__global__ void probe(Cfg c, int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x * 16; i < 160 * 1024; i += blockDim.x * 16)
        *reinterpret_cast<int4 *>(smem + i) = make_int4(0x3f803f80, 0x3f803f80, 0x3f803f80, 0x3f803f80);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t tmem = tslot;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (c.epi && threadIdx.x >= 32) {
        // warps 1-3 emulate an epilogue: tcgen05.ld 16 cols + st back, columns 256..511
        int q = (threadIdx.x >> 5) & 3;
        uint32_t lb = tmem + ((uint32_t)(q * 32) << 16) + 256;
        uint32_t r[16];
        while (!__shfl_sync(0xffffffffu, stop, 0)) {
            for (int col = 0; col < 256; col += 16) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(lb + col));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c.epi > 1) {
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                    :: "r"(lb + col), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                }
            }
        }
    }
    if (threadIdx.x < 32) {
        const uint32_t tacc = tmem + c.dcol;
        uint32_t id = idesc_bf16(128, c.N, c.a_mn, c.b_mn);
        uint32_t abase = smem_u32(smem) + c.ashift;
        uint32_t bbase = smem_u32(smem) + 96 * 1024;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            uint32_t koff = (i & 3) * 32;  // walk K inside a 128 B row for swizzled layouts
            uint64_t a = desc(abase + (c.alayout ? koff : (i & 3) * 2 * c.alab), c.alab, c.asbo, c.alayout);
            uint64_t b = desc(bbase + (c.blayout ? koff : (i & 3) * 2 * c.blbo), c.blbo, c.bsbo, c.blayout);
            asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tacc), "l"(a), "l"(b), "r"(id), "r"(1));
        }
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
        long long t1 = clock64();
        if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    // layout codes: 0 none, 2 sw128, 4 sw64, 6 sw32
    struct Named { const char *name; Cfg c; } cases[] = {
        {"none N=96 d0", {0, 0, 96, 0, 128, 256, 0, 128, 256, 0, 0, 0}},
        {"none N=96 d=416", {416, 0, 96, 0, 128, 256, 0, 128, 256, 0, 0, 0}},
        {"none N=96 d=32", {32, 0, 96, 0, 128, 256, 0, 128, 256, 0, 0, 0}},
        {"none N=96 d0 +epi ld", {0, 1, 96, 0, 128, 256, 0, 128, 256, 0, 0, 0}},
        {"none N=96 d0 +epi ld/st", {0, 2, 96, 0, 128, 256, 0, 128, 256, 0, 0, 0}},
        {"sw128 N=128 +epi ld/st", {0, 2, 128, 2, 16, 1024, 2, 16, 1024, 0, 0, 0}},
        {"sw128 N=256 d0 +epi ld/st (cols 256+ shared!)", {0, 0, 256, 2, 16, 1024, 2, 16, 1024, 0, 0, 0}},
        {"none N=32 d=64 +epi ld/st", {64, 2, 32, 0, 128, 256, 0, 128, 256, 0, 0, 0}},
    };
    const int iters = 4096;
    for (auto &cs : cases) {
        for (int grid : {1, 148}) {
            probe<<<grid, 128, 160 * 1024>>>(cs.c, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("%s: error %s\n", cs.name, cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            double cyc = (double)mx / iters;
            double floor = 128.0 * cs.c.N / 256.0;
            printf("%-42s grid=%3d  %7.1f cyc/mma  floor %5.1f  eff %5.2f\n", cs.name, grid, cyc, floor, floor / cyc);
        }
    }
    return 0;
}
