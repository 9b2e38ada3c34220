// Blackwell (sm_100a) primitives used by the tcgen05 kernels: mbarriers,
// TMA tensor loads, TMEM allocation, UMMA descriptors, tcgen05.mma / commit /
// ld.  Plain inline PTX; layouts follow the SWIZZLE_NONE ("interleaved")
// canonical UMMA layouts:
//   K-major   ((8,m),(T,2)) : ((1T,SBO),(1,LBO))   [T = 16 bytes]
//   MN-major  ((T,1,m),(8,k)) : ((1,T,SBO),(1T,LBO))
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace dp {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// 64-bit broadcast from lane 0 (makes the value provably warp-uniform for ptxas)
__device__ __forceinline__ uint64_t ushfl64(uint64_t v) {
    const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, 0);
    const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), 0);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// wait with a nanosleep back-off between polls, for warps whose waits are
// long and off the issue-critical path (so their polling leaves issue slots
// to an MMA warp on the same SM sub-partition)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAITS:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONES;\n"
        "nanosleep.u32 32;\n"
        "bra LAB_WAITS;\n"
        "DONES:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// busy-poll wait (mbarrier.test_wait never suspends the thread)
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_SPIN:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_SPIN;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- TMA -------------------------------------------------------------------
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// generic-proxy smem writes -> visible to the async proxy (UMMA operand reads)
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- TMEM ------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t addr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- UMMA ------------------------------------------------------------------
// Shared-memory matrix descriptor, SWIZZLE_NONE, sm100 version bits = 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    return d;
}

// K-major swizzled descriptor (layout 6 = SW32, 4 = SW64, 2 = SW128): 8-row
// groups SBO bytes apart, LBO unused (1).  The swizzle XOR is applied to the
// absolute shared address, so starts shifted by whole rows / 32-B K steps
// inside a 1024-B aligned box address the bytes TMA wrote there.
__device__ __forceinline__ uint64_t sdesc_sw(uint32_t saddr, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

// MN-major swizzled descriptor: MN swizzle-atom groups LBO bytes apart,
// 8-row K groups SBO bytes apart.
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                             uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> fp32, M x N.
// a_mn / b_mn select MN-major operands.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn = 0, int b_mn = 0) {
    return (1u << 4)                                  // D format f32
           | (1u << 7)                                // A bf16
           | (1u << 10)                               // B bf16
           | (static_cast<uint32_t>(a_mn) << 15)      // A major
           | (static_cast<uint32_t>(b_mn) << 16)      // B major
           | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
           | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Arrive on `bar` once every tcgen05 op issued so far by this thread completes.
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 16 consecutive fp32 columns; thread i gets lane (quarter*32 + i).
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
// 16 lanes x 4 repetitions of 128 bits (16 consecutive fp32 columns): register
// 2j + g <- lane (lane_base + lane_id / 4 + 8 g), column 4 j + lane_id % 4 (the
// fragment the wgrad transposer's 16x128b stores use, conv_tc.cu).
__device__ __forceinline__ void tmem_ld16_16x128b(uint32_t addr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x4.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}


// ---- warp-uniform issue -------------------------------------------------------
// The producer / MMA roles run their loops with the WHOLE warp converged so
// descriptors and coordinates stay in uniform registers; one elected lane
// issues the async op through a predicate inside the asm (no divergent
// branch, no per-op R2UR waterfall).  Measured: per-op issue from a
// lane-0-only branch cost ~60 cycles and made the N=96 conv MMAs 5x slower
// than the operand-bandwidth floor (scripts/umma_probe.cu).
__device__ __forceinline__ void mma_bf16_e(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_e(uint64_t *bar) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d_e(void *dst, const CUtensorMap *map, uint64_t *bar,
                                              int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
        "}\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_3d_e(void *dst, const CUtensorMap *map, uint64_t *bar,
                                              int c0, int c1, int c2) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];\n"
        "}\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// tcgen05.mma with the A operand in TMEM ("TS"): lane m = row m, a K = 16
// step = 8 consecutive 32-bit columns holding bf16 pairs (k = 2c, 2c + 1) —
// verified exactly and timed at the N/2-cycle floor by scripts/umma_ts_probe.cu.
__device__ __forceinline__ void mma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

// Eight TS MMAs over consecutive K steps (A advances 8 TMEM columns, B one
// descriptor step BSTEP per step) under ONE elect: at N <= 96 (48-cycle MMAs)
// the per-MMA elect / predicate / uniform-register setup of mma_ts_e is
// comparable to the MMA itself.  acc0 applies to the first MMA only.
template <uint32_t BSTEP>
__device__ __forceinline__ void mma_ts_x8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                          uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n"
        ".reg .pred p, q, e;\n"
        ".reg .b32 a1, a2, a3, a4, a5, a6, a7;\n"
        ".reg .b64 b1, b2, b3, b4, b5, b6, b7;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.u32 q, 1, 1;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u32 a4, %1, 32;\n"
        "add.u32 a5, %1, 40;\n"
        "add.u32 a6, %1, 48;\n"
        "add.u32 a7, %1, 56;\n"
        "add.s64 b1, %2, %5;\n"
        "add.s64 b2, %2, %6;\n"
        "add.s64 b3, %2, %7;\n"
        "add.s64 b4, %2, %8;\n"
        "add.s64 b5, %2, %9;\n"
        "add.s64 b6, %2, %10;\n"
        "add.s64 b7, %2, %11;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a4], b4, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a5], b5, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a6], b6, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a7], b7, %3, q;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc0), "n"(1 * BSTEP), "n"(2 * BSTEP), "n"(3 * BSTEP), "n"(4 * BSTEP), "n"(5 * BSTEP), "n"(6 * BSTEP), "n"(7 * BSTEP));
}

// SS form of mma_ts_x8: A and B descriptors advance ASTEP / BSTEP per K step.
template <uint32_t ASTEP, uint32_t BSTEP>
__device__ __forceinline__ void mma_bf16_x8(uint32_t d_tmem, uint64_t a, uint64_t b,
                                            uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n"
        ".reg .pred p, q, e;\n"
        ".reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.u32 q, 1, 1;\n"
        "add.s64 a1, %1, %5;\n"
        "add.s64 a2, %1, %6;\n"
        "add.s64 a3, %1, %7;\n"
        "add.s64 a4, %1, %8;\n"
        "add.s64 a5, %1, %9;\n"
        "add.s64 a6, %1, %10;\n"
        "add.s64 a7, %1, %11;\n"
        "add.s64 b1, %2, %12;\n"
        "add.s64 b2, %2, %13;\n"
        "add.s64 b3, %2, %14;\n"
        "add.s64 b4, %2, %15;\n"
        "add.s64 b5, %2, %16;\n"
        "add.s64 b6, %2, %17;\n"
        "add.s64 b7, %2, %18;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, q;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc0), "n"(1 * ASTEP), "n"(2 * ASTEP), "n"(3 * ASTEP), "n"(4 * ASTEP), "n"(5 * ASTEP), "n"(6 * ASTEP), "n"(7 * ASTEP),
        "n"(1 * BSTEP), "n"(2 * BSTEP), "n"(3 * BSTEP), "n"(4 * BSTEP), "n"(5 * BSTEP), "n"(6 * BSTEP), "n"(7 * BSTEP));
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---- CTA pairs (cta_group::2) -------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// arrive on a barrier of another CTA of the cluster (default .release.cta
// semantics, as CUTLASS's ClusterBarrier::arrive(cta_id))
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// ... with cluster-scope release: prior DSMEM stores are visible to the peer
__device__ __forceinline__ void mbar_arrive_remote_rel(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAITC:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONEC;\n"
        "bra LAB_WAITC;\n"
        "DONEC:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 16-B store into another CTA's smem that performs complete_tx(16) on that
// CTA's mbarrier when it lands (no release fence on the issuing thread)
__device__ __forceinline__ void st_async_v4(uint32_t cluster_addr, uint4 v, uint32_t cluster_bar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
            cluster_addr),
        "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(cluster_bar)
        : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t cluster_addr, uint4 v) {
    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(cluster_addr), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
// Out-of-line allocation: an inlined `.sync.aligned` tcgen05.alloc inside a
// role branch makes ptxas treat the whole kernel as possibly non-converged,
// and every tcgen05.mma then goes through an ELECT / R2UR.BROADCAST /
// VOTEU sequence (~15 instructions per MMA on the single issuing warp).
// Behind a call the MMA warp's descriptor math stays on the uniform datapath
// (measured in SASS: 122 -> 23 R2UR, 51 -> 3 ELECT for 27 MMAs).
static __device__ __noinline__ void tmem_alloc_ool(uint32_t *dst, uint32_t ncols) { tmem_alloc(dst, ncols); }
static __device__ __noinline__ void tmem_alloc2_ool(uint32_t *dst, uint32_t ncols) { tmem_alloc2(dst, ncols); }
__device__ __forceinline__ void tmem_dealloc2(uint32_t addr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(ncols));
}
// M = 256 MMA over the CTA pair (A rows and B columns split between the two
// CTAs' shared memory at the same offsets; D rows in each CTA's TMEM).
// Issued by the even CTA only.
__device__ __forceinline__ void mma2_bf16_e(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// Three cta_group::2 MMAs into the same accumulator under ONE elect, the
// second and third at fixed descriptor offsets (DA, DB in 16-B units): the kw
// taps of a merged conv step.  Cuts the per-MMA issue work (elect, votes,
// uniform-register moves) the single-MMA helper pays three times.
template <uint32_t DA, uint32_t DB>
__device__ __forceinline__ void mma2_bf16_x3(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        ".reg .b64 a1, a2, b1, b2;\n"
        "setp.eq.u32 p, 1, 1;\n"
        "add.s64 a1, %1, %4;\n"
        "add.s64 a2, %1, %5;\n"
        "add.s64 b1, %2, %6;\n"
        "add.s64 b2, %2, %7;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "n"(DA), "n"(2 * DA), "n"(DB), "n"(2 * DB));
}
// As mma2_bf16_x3 / mma_bf16_x3 with the A descriptor split into its low
// word (start address + LBO: the only part a K step or kw tap moves) and its
// constant high word: the per-MMA A arithmetic is one 32-bit add instead of
// a 64-bit add pair, and the high word stays in one uniform register.
template <uint32_t DA, uint32_t DB, bool PAIR>
__device__ __forceinline__ void mma_bf16_x3_lo(uint32_t d_tmem, uint32_t alo, uint32_t ahi,
                                               uint64_t b, uint32_t idesc) {
    if constexpr (PAIR)
        asm volatile(
            "{\n"
            ".reg .pred p, e;\n"
            ".reg .b32 l1, l2;\n"
            ".reg .b64 a0, a1, a2, b1, b2;\n"
            "setp.eq.u32 p, 1, 1;\n"
            "add.u32 l1, %1, %5;\n"
            "add.u32 l2, %1, %6;\n"
            "mov.b64 a0, {%1, %2};\n"
            "mov.b64 a1, {l1, %2};\n"
            "mov.b64 a2, {l2, %2};\n"
            "add.s64 b1, %3, %7;\n"
            "add.s64 b2, %3, %8;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a0, %3, %4, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %4, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %4, p;\n"
            "}\n" ::"r"(d_tmem),
            "r"(alo), "r"(ahi), "l"(b), "r"(idesc), "n"(DA), "n"(2 * DA), "n"(DB), "n"(2 * DB));
    else
        asm volatile(
            "{\n"
            ".reg .pred p, e;\n"
            ".reg .b32 l1, l2;\n"
            ".reg .b64 a0, a1, a2, b1, b2;\n"
            "setp.eq.u32 p, 1, 1;\n"
            "add.u32 l1, %1, %5;\n"
            "add.u32 l2, %1, %6;\n"
            "mov.b64 a0, {%1, %2};\n"
            "mov.b64 a1, {l1, %2};\n"
            "mov.b64 a2, {l2, %2};\n"
            "add.s64 b1, %3, %7;\n"
            "add.s64 b2, %3, %8;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, %3, %4, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %4, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %4, p;\n"
            "}\n" ::"r"(d_tmem),
            "r"(alo), "r"(ahi), "l"(b), "r"(idesc), "n"(DA), "n"(2 * DA), "n"(DB), "n"(2 * DB));
}
// cta_group::1 form of mma2_bf16_x3.
template <uint32_t DA, uint32_t DB>
__device__ __forceinline__ void mma_bf16_x3(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        ".reg .b64 a1, a2, b1, b2;\n"
        "setp.eq.u32 p, 1, 1;\n"
        "add.s64 a1, %1, %4;\n"
        "add.s64 a2, %1, %5;\n"
        "add.s64 b1, %2, %6;\n"
        "add.s64 b2, %2, %7;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "n"(DA), "n"(2 * DA), "n"(DB), "n"(2 * DB));
}
// commit: arrive on `bar` (same offset) in both CTAs of the pair
__device__ __forceinline__ void mma2_commit_mc_e(uint64_t *bar) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        ".reg .b16 m;\n"
        "mov.b16 m, 3;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}
// TMA load into this CTA's smem whose complete_tx lands on the EVEN CTA's
// barrier at the same offset (both CTAs of a pair feed one MMA).
__device__ __forceinline__ void tma_load_5d_2sm_e(void *dst, const CUtensorMap *map,
                                                  uint32_t leader_bar, int c0, int c1, int c2,
                                                  int c3, int c4) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
        "}\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(leader_bar)
        : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}

}  // namespace tc

// host: cuTensorMapEncodeTiled through the runtime's driver entry point
// (no -lcuda link dependency).
int encode_tensor_map(CUtensorMap *map, CUtensorMapDataType dtype, int rank, void *base,
                      const uint64_t *dims, const uint64_t *strides_bytes, const uint32_t *box,
                      CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE);

}  // namespace dp
