// tcgen05 + TMA implicit-GEMM convolution (bf16 in, fp32 accumulate in TMEM)
// for channels-last activations, stride 1 — the forward conv and, through a
// flipped/transposed weight image, the data gradient.
//
// GEMM view: M = 128 output voxels along W (one TMEM lane each), N = C_out
// (TMEM columns), K = taps x C_in (16 channels per tcgen05.mma).
//
// Geometry roles.  Spatial dims are mapped onto (P, Q, W):
//   3-D (D,H,W): P = D, Q = H;   2-D (H,W): P = 1 (dummy), Q = H.
// A work unit is a column (b, p_out, 128-voxel W tile) and a chunk of
// output rows q_out in [q0, q1).  The unit streams INPUT rows q_in along Q;
// one pipeline stage holds the KP input rows (kp = 0..KP-1) at one q_in
// for all C_in, staged by TMA as 8-channel "chunk planes": plane = 130
// voxels x 16 B, so shifting the UMMA A descriptor by 16 B shifts the
// window by one voxel (the kw taps reuse the same smem; TMA zero-fills
// every out-of-range voxel = the conv padding).  Each staged row feeds the
// KQ output rows it contributes to (q_out = q_in - base_q - kq).  Their
// fp32 accumulators sit in a ring of TMEM slots laid out in DECREASING
// column order (slot(r) = (NSLOT-1 - r mod NSLOT) * N), so the KQ rows a
// staged input row feeds are adjacent columns [row j | row j-1 | row j-2]:
// ONE tcgen05.mma with N = KQ*C_out (B rows ordered (kq, c_out)) performs
// all KQ tap contributions of a (kp, kw, 16-channel) step.  Slots are zeroed
// by the epilogue when it drains them, so every MMA accumulates.  Input rows
// are loaded once per unit instead of KQ times, and each A tile is read once
// per KQ*C_out columns (3x fewer smem operand bytes and MMA issues than a
// per-tap N = C_out GEMM).
//
// Virtual halo block: on the sharded dim (P for 3-D, Q for 2-D) input rows
// [0, main) come from the local block's tensor map and [main, main+halo)
// from the received halo's map; anything else is out of bounds -> zeros.
// That is the reference's trimmed + zero-padded extended block
// (domainpar/ops.py:397-413) without ever materialising it.
//
// Warp roles (192 threads, one CTA per SM, persistent over units):
//   warp 0     TMA producer (one lane)          smem ring: full/empty mbarriers
//   warp 1     tcgen05.mma issuer (one lane)    TMEM ring: tfull/tempty mbarriers
//   warps 2-5  epilogue: tcgen05.ld -> bf16 -> 16-B global stores
#include "tc_common.cuh"
#include <type_traits>

namespace dp {
namespace {

constexpr int kTileW = 128;
constexpr int kThreads = 192;

// Channel blocking of the activation operand: one TMA box per (input row,
// channel block) = BW voxels x cblk channels, i.e. a single contiguous run
// of BW * cblk * 2 bytes in a channels-last tensor, landed with the matching
// hardware swizzle (32/64/128 B rows).  The UMMA A operand is that box read
// K-major-swizzled; the kw taps are descriptor shifts of one row
// (rowbytes) — the swizzle is a function of the absolute smem address, so a
// shifted start reads the same bytes TMA wrote.
__host__ __device__ constexpr int chan_block(int c) {
    return c == 16 ? 16 : c == 32 ? 32 : (c % 64 == 0 ? 64 : 16);
}
__host__ __device__ constexpr uint32_t swz_layout(int cblk) {  // UMMA layout_type field
    return cblk == 16 ? 6u : cblk == 32 ? 4u : 2u;            // SW32 / SW64 / SW128
}
__host__ __device__ constexpr int box_bytes(int cblk, int kw) {
    return (((kTileW + kw - 1) * cblk * 2) + 1023) / 1024 * 1024;
}

struct ConvTcParams {
    int B, Cin, Cout;
    int Pin, Qin, Win;        // main-block input extents (P, Q, W roles)
    int Pout, Qout, Wout;     // output extents
    int KP, KQ, KW;
    int base_p, base_q, base_w;
    int split;                // 0: halo on P, 1: halo on Q, -1: none
    int halo;                 // halo rows on the split dim
    __nv_bfloat16 *y, *y2;    // output / output rows >= ysplit on the split dim
    int64_t ys[4], y2s[4];    // element strides (b, p, q, w); channel stride 1
    int ysplit_dim, ysplit;   // -1: none
    int n_wt, q_chunk, n_qc, n_units;
    int nstage;               // pipeline depth
    int wimg_bytes;
    const __nv_bfloat16 *wimg;
    int dbg;                  // profiling ablations (DP_CONV_DBG): 1 no stores, 2 no MMA, 4 no TMA
    float *yf, *yf2;          // fp32 outputs (the bf16x3 fp32 path) instead of y / y2
    int64_t ycs, y2cs;        // their channel strides (elements)
    int qorg;                 // global index of output row q = 0 (ring alignment)
    int cperm;                // bf16 output through the coalesced drain (permuted B columns)
    int Pu;                   // units along P: ceil(Pout / PPN)
};

// Template arguments KP_/KQ_/KW_/CIN_ = 0 select the runtime-shaped kernel;
// non-zero values give the fully unrolled MMA issue the hot shapes use (a
// runtime-bounded loop costs ~180 issue cycles per MMA vs ~56 of operand
// time for N=96 — measured, scripts/umma_probe2.cu).
// PAIR: the CTA pair of a (2,1,1) cluster runs M = 256 tcgen05.mma.cta_group::2
// over two adjacent 128-voxel W tiles (CTA r holds tile 2 wp + r: its A rows,
// its half of the B columns, its D rows); only the even CTA issues MMAs.  Per
// CTA an N = 96 MMA then reads 4 KB of A + 1.5 KB of B (compute-bound, 48
// cycles) instead of 4 KB + 3 KB (shared-memory-bound, 56 cycles).
// TMEM accumulator ring.  NSLOT logical row slots of N columns, slot(r) =
// NSLOT-1 - r mod NSLOT, plus (N <= 64) two EXTENSION slots after the ring:
// the merged MMA of a top row near the ring's end writes the KQ-1 <= 2 rows
// that wrapped past column (NSLOT-1)*N into the extension slots instead
// (row slot L in {0, 1} -> column (NSLOT + L)*N), so EVERY interior stage is
// one merged N = KQ*C_out MMA per (kp, kw, kc).  The epilogue adds the
// extension slot into rows L in {0, 1} and zeroes both.  (Without the
// extension 2 of every 16 rows fell back to per-kq MMAs with the full A
// operand re-read per kq: +14 % stage time for N = 96, +21 % for N = 48.)
__host__ __device__ constexpr bool ring_ext(int N, int cols = 512) { return cols / N >= 8; }
__host__ __device__ constexpr int ring_slots(int N, int cols = 512) {
    return ring_ext(N, cols) ? ((cols / N) < 18 ? (cols / N) : 18) - 2
                             : ((cols / N) < 16 ? (cols / N) : 16);
}

// X3: the bf16x3 fp32 path.  The MMA contracts over CIN_ = 6 C channel blocks
// [xh xh xh xm xm xl] (against W' = [wh wm wl wh wm wh], conv_x3.cu) but the
// activation holds each part ONCE, as batch blocks [part][B][..][C] (the
// layout the TS wgrad reads too, so one split serves fwd/dgrad and wgrad):
// the producer loads the 3 part boxes of a row (batch coordinate
// part * B + b), and K block b reads part x3_part(b) — half the split writes
// and TMA bytes of a materialised 6-block operand.
__host__ __device__ constexpr int x3_part(int blk) { return blk < 3 ? 0 : blk < 5 ? 1 : 2; }

// PPN = 2 (P-pair): a unit covers two adjacent output planes.  A stage holds
// the KP + 1 input rows the two planes need (plane t reads boxes t .. t+KP-1),
// each plane accumulates in its own TMEM ring (columns [t * 256, +256)), and
// the epilogue drains both rows of a slot.  Every input row then crosses
// L2 -> SMEM (KP + 1) / 2 times per plane instead of KP: the TMA input stream
// the ablations price at ~0.1 ms per fwd / dgrad kernel.  The MMAs, their
// order per plane and the ring / extension-slot mapping are those of PPN = 1.
template <int N, int KP_, int KQ_, int KW_, int CIN_, bool PAIR = false, bool X3 = false,
          int PPN = 1>
__global__ void __launch_bounds__(kThreads, 1)
conv_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
               const ConvTcParams p) {
    using namespace tc;
    extern __shared__ __align__(1024) uint8_t smem[];
    // warp index through a shuffle: ptxas then knows it is warp-uniform, the
    // role branches stay on the uniform datapath and the MMA warp computes its
    // descriptors in uniform registers (no per-MMA ELECT + R2UR.BROADCAST:
    // ~15 -> ~4 instructions per tcgen05.mma, the issue rate that bounded
    // the small-N stages)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? __shfl_sync(0xffffffffu, cluster_ctarank(), 0) : 0u;
    const int u0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;          // first unit
    const int ustep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    constexpr bool kStatic = KP_ > 0;
    const int KP = kStatic ? KP_ : p.KP;
    const int KQ = kStatic ? KQ_ : p.KQ;
    const int KW = kStatic ? KW_ : p.KW;
    const int CIN = kStatic ? CIN_ : p.Cin;
    static_assert(!X3 || (KP_ > 0 && CIN_ % 96 == 0), "X3: static 6-block shapes only");
    static_assert(PPN == 1 || (KP_ > 0 && KW_ == 3 && !X3), "PPN = 2: static 3-tap shapes only");
    constexpr int RCOLS = 512 / PPN;         // TMEM columns of one plane's ring
    const int CBLK = X3 ? CIN / 6 : chan_block(CIN);
    const int NBLK = X3 ? 3 : CIN / CBLK;
    const int KPB = CBLK / 16;               // 16-channel MMA steps per block row
    const int KC = CIN / 16;
    const int ROWB = CBLK * 2;               // bytes per voxel row of a box
    const int BOXB = box_bytes(CBLK, KW);
    constexpr int NSLOT = ring_slots(N, RCOLS);
    constexpr bool EXT = ring_ext(N, RCOLS);
    constexpr int NPHYS = EXT ? NSLOT + 2 : NSLOT;
    const bool wrap_ok = EXT && KQ <= 3;     // wrapped rows go to the extension slots
    const int BW = kTileW + KW - 1;
    const int NROW = KP + PPN - 1;           // input rows (boxes per channel block) per stage
    const uint32_t stage_bytes = (uint32_t)(NROW * NBLK * BOXB);

    uint8_t *wsm = smem;
    uint8_t *stages = smem + ((p.wimg_bytes + 1023) & ~1023);
    uint64_t *bars = reinterpret_cast<uint64_t *>(stages + (size_t)p.nstage * stage_bytes);
    uint64_t *full = bars, *empty = bars + p.nstage;
    uint64_t *tfull = empty + p.nstage, *tempty = tfull + NSLOT;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + NSLOT);

    // weights: global image -> smem once per CTA (generic proxy), then fence
    // (PAIR: this CTA's half of the B columns, image [rank][...])
    const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(p.wimg) + (size_t)rank * p.wimg_bytes;
    for (int i = threadIdx.x * 16; i < p.wimg_bytes; i += kThreads * 16)
        *reinterpret_cast<int4 *>(wsm + i) = *reinterpret_cast<const int4 *>(wsrc + i);
    fence_async_smem();
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < p.nstage; ++i) {
                mbar_init(&full[i], 1);
                mbar_init(&empty[i], 1);
            }
            for (int i = 0; i < NSLOT; ++i) {
                mbar_init(&tfull[i], 1);
                mbar_init(&tempty[i], PAIR ? 8 : 128);   // PAIR: one arrival per warp x 2 CTAs
            }
            mbar_fence_init();
            tma_prefetch(&xmap);
            tma_prefetch(&hmap);
        }
        __syncwarp();
        if constexpr (PAIR) tmem_alloc2_ool(tmem_slot, 512);
        else tmem_alloc_ool(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);   // uniform for ptxas
    if (warp >= 2) {
        // every accumulator slot starts at zero (MMAs always accumulate)
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        for (int t = 0; t < PPN; ++t)
            for (int c = 0; c < NPHYS * N; c += 16) tmem_st16(lane_base + t * RCOLS + c, z);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();
    tc_fence_after();

    if (warp == 0) {
        // ===================== TMA producer (whole warp, elected issue) =====================
        const uint32_t lead_full = PAIR ? mapa_shared(smem_u32(full), 0) : 0u;
        uint32_t it = 0, idx = 0, ph = 0;
        for (int u = u0; u < p.n_units; u += ustep) {
            int r = u;
            const int wt = PAIR ? (r % p.n_wt) * 2 + (int)rank : r % p.n_wt; r /= p.n_wt;
            const int qc = r % p.n_qc; r /= p.n_qc;
            const int po = (r % p.Pu) * PPN;    // first output plane of the unit
            const int b = r / p.Pu;
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int nrows = (q1 - q0) + KQ - 1;
            const int wc = p.base_w + wt * kTileW;
            for (int s = 0; s < nrows;
                 ++s, ++it, (++idx == (uint32_t)p.nstage ? (idx = 0u, ph ^= 1u) : 0u)) {
                mbar_wait(&empty[idx], ph ^ 1);
                if (p.dbg & 4) {
                    if (lane == 0) mbar_arrive(&full[idx]);
                    __syncwarp();
                    continue;
                }
                if (!PAIR || rank == 0)
                    mbar_expect_tx_e(&full[idx], (uint32_t)((PAIR ? 2 : 1) * NROW * NBLK * BW * ROWB));
                uint8_t *dst = stages + (size_t)idx * stage_bytes;
                const int qv = p.base_q + q0 + s;
                for (int kp = 0; kp < NROW; ++kp) {   // input rows po + 0 .. po + NROW - 1
                    const int pv = p.base_p + po + kp;
                    const CUtensorMap *map = &xmap;
                    int pc = pv, qcrd = qv;
                    if (p.split == 0 && pv >= p.Pin && pv < p.Pin + p.halo) {
                        map = &hmap;
                        pc = pv - p.Pin;
                    } else if (p.split == 1 && qv >= p.Qin && qv < p.Qin + p.halo) {
                        map = &hmap;
                        qcrd = qv - p.Qin;
                    }
                    for (int cb = 0; cb < NBLK; ++cb) {
                        if constexpr (PAIR)
                            tma_load_5d_2sm_e(dst + (size_t)(kp * NBLK + cb) * BOXB, map,
                                              lead_full + idx * 8, X3 ? 0 : cb * CBLK, wc, qcrd,
                                              pc, X3 ? cb * p.B + b : b);
                        else
                            tma_load_5d_e(dst + (size_t)(kp * NBLK + cb) * BOXB, map, &full[idx],
                                          X3 ? 0 : cb * CBLK, wc, qcrd, pc, X3 ? cb * p.B + b : b);
                    }
                }
            }
        }
    } else if (warp == 1 && (!PAIR || rank == 0)) {
        // ===================== MMA issuer (whole warp, elected issue) =====================
        const uint32_t idesc_one = idesc_bf16(PAIR ? 256 : 128, N);
        const uint32_t idesc_all = idesc_bf16(PAIR ? 256 : 128, N * KQ);
        // B blocks: single CTA: (kp,kw,kc) blocks of KQ*N rows (the per-kq MMAs use row
        // slices); PAIR: this CTA's halves — merged blocks of KQ*N/2 rows, then per-kq
        // blocks of N/2 rows (the two MMA shapes split their columns differently)
        const uint32_t blk = PAIR ? (uint32_t)KQ * N * 16 : (uint32_t)KQ * N * 32;
        const uint32_t kqblk0 = (uint32_t)(KP * KW * KC) * blk, kqblk = (uint32_t)N * 16;
        const uint64_t bdesc0 = sdesc(smem_u32(wsm), 128, 256);
        const uint64_t adesc0 = sdesc_sw(smem_u32(stages), 8 * ROWB, swz_layout(CBLK));
        auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
            if constexpr (PAIR) mma2_bf16_e(d, a, b, id, 1u);
            else mma_bf16_e(d, a, b, id, 1u);
        };
        auto commit = [&](uint64_t *bar) {
            if constexpr (PAIR) mma2_commit_mc_e(bar);
            else mma_commit_e(bar);
        };
        // stage slot / phase carried across iterations: no integer division per
        // stage (measured: L1 dgrad 0.600 -> 0.536 ms, L1 fwd 0.512 -> 0.494)
        uint32_t it = 0, row_base = 0, idx = 0, ph = 0;
        for (int u = u0; u < p.n_units; u += ustep) {
            int r = u / p.n_wt;
            const int qc = r % p.n_qc;
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int nq = q1 - q0;
            const int nrows = nq + KQ - 1;
            if (wrap_ok) {
                // ring slot of output row q = (global q) mod NSLOT: every row splits
                // between ring and extension slot exactly as in any other launch
                // (sharded or not), so the sums are bitwise sharding-invariant.
                // Skipped slots pass through empty (tempty -> tfull, no MMA).
                const uint32_t pad = (uint32_t)(((q0 + p.qorg - (int)(row_base % NSLOT)) % NSLOT +
                                                 NSLOT) % NSLOT);
                for (uint32_t d = 0; d < pad; ++d, ++row_base) {
                    mbar_wait(&tempty[row_base % NSLOT], ((row_base / NSLOT) & 1) ^ 1);
                    commit(&tfull[row_base % NSLOT]);
                }
            }
            for (int s = 0; s < nrows;
                 ++s, ++it, (++idx == (uint32_t)p.nstage ? (idx = 0u, ph ^= 1u) : 0u)) {
                if (s < nq) {
                    // row s starts here: its slot must have been drained + zeroed
                    const uint32_t row = row_base + s;
                    mbar_wait(&tempty[row % NSLOT], ((row / NSLOT) & 1) ^ 1);
                }
                mbar_wait(&full[idx], ph);
                tc_fence_after();
                const uint64_t adesc = adesc0 + ((idx * stage_bytes) >> 4);
                const uint32_t top = row_base + s;  // row fed through kq = 0
                const bool merged =
                    s >= KQ - 1 && s < nq && (wrap_ok || (int)(top % NSLOT) >= KQ - 1);
                if (p.dbg & 2) {
                } else if (kStatic && KW_ == 3 && (X3 || PPN > 1 || !(p.dbg & (16 | 32)))) {
                    // the three kw taps of each (kp, kc) issued as one group (one elect;
                    // measured 4-7 % faster than one elect per MMA)
                    constexpr int CS = CIN_ > 0 ? CIN_ : 16, KQS = KQ_ > 0 ? KQ_ : 1;
                    constexpr int CB = X3 ? CS / 6 : chan_block(CS), NB = X3 ? 3 : CS / CB;
                    constexpr int KPB_S = CB / 16, KC_S = CS / 16;
                    // K step kc -> stored 16-channel step (X3: part of its 6-block index)
                    auto kstore = [](int kc) {
                        return X3 ? x3_part(kc / KPB_S) * KPB_S + kc % KPB_S : kc;
                    };
                    constexpr uint32_t DA = (uint32_t)(CB * 2) >> 4;                     // one voxel row
                    constexpr uint32_t BLK = PAIR ? KQS * N * 16 : KQS * N * 32;        // == blk
                    constexpr uint32_t DBM = (uint32_t)(KC_S * BLK) >> 4;                // kw step, merged
                    constexpr uint32_t DBQ = PAIR ? (uint32_t)(KC_S * KQS * N * 16) >> 4 : DBM;  // per-kq
                    const uint32_t ahi = (uint32_t)(adesc >> 32), alo = (uint32_t)adesc;
                    auto grp = [&](uint32_t d, uint32_t aoff16, uint64_t b, uint32_t id, auto dbt) {
                        constexpr uint32_t DBV = decltype(dbt)::value;
                        mma_bf16_x3_lo<DA, DBV, PAIR>(d, alo + aoff16, ahi, b, id);
                    };
                    // plane t of the unit: its own ring, input boxes t .. t + KP - 1
#pragma unroll
                    for (int t = 0; t < PPN; ++t) {
                    if (merged) {
                        const uint32_t d = tmem + t * RCOLS + (NSLOT - 1 - top % NSLOT) * N;
#pragma unroll
                        for (int kp = 0; kp < KP; ++kp)
#pragma unroll
                            for (int kc = 0; kc < KC_S; ++kc) {
                                const uint32_t aoff = ((t + kp) * NB + kstore(kc) / KPB_S) * BOXB + (kstore(kc) % KPB_S) * 32;
                                const uint32_t boff = ((kp * 3) * KC_S + kc) * BLK;
                                grp(d, aoff >> 4, bdesc0 + (boff >> 4), idesc_all,
                                    std::integral_constant<uint32_t, DBM>{});
                            }
                    } else {
#pragma unroll
                        for (int kq = 0; kq < KQS; ++kq) {
                            const int j = s - kq;
                            if (j < 0 || j >= nq) continue;
                            const uint32_t row = row_base + j;
                            // the column the merged MMA of this top row would use (ring or
                            // extension slot): identical sums whichever MMA form adds them
                            const uint32_t d = tmem + t * RCOLS +
                                               (wrap_ok ? NSLOT - 1 - top % NSLOT + kq
                                                        : NSLOT - 1 - row % NSLOT) * N;
#pragma unroll
                            for (int kp = 0; kp < KP; ++kp)
#pragma unroll
                                for (int kc = 0; kc < KC_S; ++kc) {
                                    const uint32_t aoff = ((t + kp) * NB + kstore(kc) / KPB_S) * BOXB + (kstore(kc) % KPB_S) * 32;
                                    const uint32_t boff =
                                        PAIR ? kqblk0 + (((kp * 3) * KC_S + kc) * KQS + kq) * kqblk
                                             : ((kp * 3) * KC_S + kc) * BLK + kq * (N / 8) * 256;
                                    grp(d, aoff >> 4, bdesc0 + (boff >> 4), idesc_one,
                                        std::integral_constant<uint32_t, DBQ>{});
                                }
                        }
                    }
                    }   // planes t
                } else if (merged) {
                    const uint32_t d = tmem + (NSLOT - 1 - top % NSLOT) * N;
#pragma unroll
                    for (int kp = 0; kp < KP; ++kp)
#pragma unroll
                        for (int kw = 0; kw < KW; ++kw)
#pragma unroll
                            for (int kc = 0; kc < KC; ++kc) {
                                const uint32_t aoff = (kp * NBLK + kc / KPB) * BOXB +
                                                      ((p.dbg & 16) ? kw * 8 * ROWB : kw * ROWB) +
                                                      (kc % KPB) * 32;
                                const uint32_t boff = ((kp * KW + kw) * KC + kc) * blk;
                                mma(d, adesc + (aoff >> 4), bdesc0 + (boff >> 4), idesc_all);
                            }
                } else {
#pragma unroll
                    for (int kq = 0; kq < KQ; ++kq) {
                        const int j = s - kq;
                        if (j < 0 || j >= nq) continue;
                        const uint32_t row = row_base + j;
                        // the column the merged MMA of this top row would use (ring or
                            // extension slot): identical sums whichever MMA form adds them
                            const uint32_t d = tmem + (wrap_ok ? NSLOT - 1 - top % NSLOT + kq
                                                               : NSLOT - 1 - row % NSLOT) * N;
#pragma unroll
                        for (int kp = 0; kp < KP; ++kp)
#pragma unroll
                            for (int kw = 0; kw < KW; ++kw)
#pragma unroll
                                for (int kc = 0; kc < KC; ++kc) {
                                    const uint32_t aoff = (kp * NBLK + kc / KPB) * BOXB +
                                                          kw * ROWB + (kc % KPB) * 32;
                                    const uint32_t boff =
                                        PAIR ? kqblk0 + (((kp * KW + kw) * KC + kc) * KQ + kq) * kqblk
                                             : ((kp * KW + kw) * KC + kc) * blk +
                                                   kq * (N / 8) * 256;
                                    mma(d, adesc + (aoff >> 4), bdesc0 + (boff >> 4), idesc_one);
                                }
                    }
                }
                commit(&empty[idx]);
                const int jd = s - (KQ - 1);
                if (jd >= 0 && jd < nq) commit(&tfull[(row_base + jd) % NSLOT]);
            }
            row_base += nq;
        }
    } else if (warp >= 2) {
        // ===================== epilogue =====================
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;  // TMEM lane = voxel within the tile
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t lead_tempty = PAIR ? mapa_shared(smem_u32(tempty), 0) : 0u;
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        // ring slot / phase of the next row to drain (division-free, as the MMA loop)
        uint32_t eslot = 0, eph = 0;
        auto next_row = [&]() {
            if (++eslot == (uint32_t)NSLOT) { eslot = 0; eph ^= 1u; }
        };
        auto free_slot = [&](uint32_t slot) {
            if constexpr (PAIR) {
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) mbar_arrive(&tempty[slot]);
                    else mbar_arrive_remote(lead_tempty + slot * 8);
                }
            } else {
                mbar_arrive(&tempty[slot]);
            }
        };
        // bf16 output through the coalesced drain (fp32 outputs / ablations take the
        // per-lane path below); the halo output part must share the W stride
        const bool fast = p.cperm && (PPN > 1 || !(p.dbg & 8));   // PPN = 2: always
        for (int u = u0; u < p.n_units; u += ustep) {
            int r = u;
            const int wt = PAIR ? (r % p.n_wt) * 2 + (int)rank : r % p.n_wt; r /= p.n_wt;
            const int qc = r % p.n_qc; r /= p.n_qc;
            const int po = (r % p.Pu) * PPN;    // first output plane of the unit
            const int b = r / p.Pu;
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int w = wt * kTileW + m;
            if (wrap_ok) {   // the MMA warp's alignment rows: drain nothing, free the slot
                const uint32_t pad = (uint32_t)(((q0 + p.qorg - (int)eslot) % NSLOT + NSLOT) % NSLOT);
                for (uint32_t d = 0; d < pad; ++d) {
                    mbar_wait_sleep(&tfull[eslot], eph);
                    free_slot(eslot);
                    next_row();
                }
            }
            if (fast) {
                // bf16 output, coalesced: 16x128b loads give thread t the columns
                // 4 jj + t%4 of voxels 16 h + 8 g + t/4 of this warp's quarter; the B
                // columns are permuted (conv_tc_weight_image*, cperm) so those are
                // channels U (4 k + t%4) + i (jj = k U + i): each of the 4 threads of a
                // voxel holds whole U-channel chunks, and one store instruction writes
                // 8 voxels x 4 chunks = 8 contiguous runs of 4 U bf16 (512 B for N = 32)
                // instead of 32 half-used sectors per instruction.  Addresses are set
                // up once per unit: a row pointer advanced by the Q stride (switching
                // to the halo output at the split row) + 4 per-voxel offsets.
                constexpr int NJ = N / 4, U = (N % 32 == 0) ? 8 : 4;
                // per plane of the unit: row pointer, Q step, split row (Q-split halo
                // output), and whether the plane exists (an odd P extent's last pair)
                __nv_bfloat16 *rowp[PPN], *rowp2[PPN];
                int64_t rstep[PPN];
                int jsw[PPN];
                bool pok[PPN];
#pragma unroll
                for (int t = 0; t < PPN; ++t) {
                    const int pl = po + t;
                    pok[t] = pl < p.Pout;
                    jsw[t] = 1 << 30;
                    rowp2[t] = nullptr;
                    if (p.ysplit_dim == 0 && pl >= p.ysplit) {
                        rowp[t] = p.y2 + b * p.y2s[0] + (int64_t)(pl - p.ysplit) * p.y2s[1] +
                                  (int64_t)q0 * p.y2s[2];
                        rstep[t] = p.y2s[2];
                    } else {
                        rowp[t] = p.y + b * p.ys[0] + (int64_t)pl * p.ys[1] + (int64_t)q0 * p.ys[2];
                        rstep[t] = p.ys[2];
                        if (p.ysplit_dim == 1) {
                            jsw[t] = max(0, p.ysplit - q0);
                            rowp2[t] = p.y2 + b * p.y2s[0] + (int64_t)pl * p.y2s[1] +
                                       (int64_t)(q0 + jsw[t] - p.ysplit) * p.y2s[2];
                        }
                    }
                }
                int off[2][2];
                bool ok[2][2];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
                        const int wv = wt * kTileW + quarter * 32 + 16 * h + 8 * g + (lane >> 2);
                        ok[h][g] = wv < p.Wout && !(p.dbg & 1);
                        off[h][g] = wv * (int)p.ys[3] + U * (lane & 3);
                    }
                for (int j = 0; j < q1 - q0; ++j) {
                    const uint32_t slot = eslot;
                    mbar_wait_sleep(&tfull[slot], eph);
                    next_row();
                    tc_fence_after();
                    uint32_t v[PPN][2][2][NJ];
#pragma unroll
                    for (int t = 0; t < PPN; ++t) {
                        const uint32_t col = lane_base + t * RCOLS + (NSLOT - 1 - slot) * N;
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int c0 = 0; c0 < N; c0 += 16) {
                                uint32_t tt[8];
                                tmem_ld16_16x128b(col + ((uint32_t)(16 * h) << 16) + c0, tt);
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj) {
                                    v[t][h][0][c0 / 4 + jj] = tt[2 * jj];
                                    v[t][h][1][c0 / 4 + jj] = tt[2 * jj + 1];
                                }
                            }
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < N; c += 16) tmem_st16(col + c, z);
                        if (wrap_ok && slot >= (uint32_t)(NSLOT - 2)) {
                            const uint32_t ecol =
                                lane_base + t * RCOLS + (uint32_t)(2 * NSLOT - 1 - slot) * N;
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int c0 = 0; c0 < N; c0 += 16) {
                                    uint32_t tt[8];
                                    tmem_ld16_16x128b(ecol + ((uint32_t)(16 * h) << 16) + c0, tt);
                                    tmem_wait_ld();
#pragma unroll
                                    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                                        for (int g = 0; g < 2; ++g)
                                            v[t][h][g][c0 / 4 + jj] = __float_as_uint(
                                                __uint_as_float(v[t][h][g][c0 / 4 + jj]) +
                                                __uint_as_float(tt[2 * jj + g]));
                                }
#pragma unroll
                            for (int c = 0; c < N; c += 16) tmem_st16(ecol + c, z);
                        }
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    free_slot(slot);
#pragma unroll
                    for (int t = 0; t < PPN; ++t) {
                        if (j == jsw[t]) {
                            rowp[t] = rowp2[t];
                            rstep[t] = p.y2s[2];
                        }
                        if (!pok[t]) continue;
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int g = 0; g < 2; ++g) {
                                __nv_bfloat16 *dst = rowp[t] + off[h][g];
#pragma unroll
                                for (int k = 0; k < NJ / U; ++k) {
                                    const uint32_t *a = &v[t][h][g][k * U];
                                    if constexpr (U == 8) {
                                        uint4 pk;
                                        pk.x = pack_bf16(__uint_as_float(a[0]), __uint_as_float(a[1]));
                                        pk.y = pack_bf16(__uint_as_float(a[2]), __uint_as_float(a[3]));
                                        pk.z = pack_bf16(__uint_as_float(a[4]), __uint_as_float(a[5]));
                                        pk.w = pack_bf16(__uint_as_float(a[6]), __uint_as_float(a[7]));
                                        if (ok[h][g]) *reinterpret_cast<uint4 *>(dst + 4 * U * k) = pk;
                                    } else {
                                        uint2 pk;
                                        pk.x = pack_bf16(__uint_as_float(a[0]), __uint_as_float(a[1]));
                                        pk.y = pack_bf16(__uint_as_float(a[2]), __uint_as_float(a[3]));
                                        if (ok[h][g]) *reinterpret_cast<uint2 *>(dst + 4 * U * k) = pk;
                                    }
                                }
                            }
                        rowp[t] += rstep[t];
                    }
                }
                continue;
            }
            for (int j = 0; j < q1 - q0; ++j) {
                const uint32_t slot = eslot;
                mbar_wait_sleep(&tfull[slot], eph);
                next_row();
                tc_fence_after();
                const uint32_t col = lane_base + (NSLOT - 1 - slot) * N;
                uint32_t v[N];
                if (!(p.dbg & 8)) {
#pragma unroll
                for (int c = 0; c < N; c += 16) {
                    uint32_t t[16];
                    tmem_ld16(col + c, t);
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[c + i] = t[i];
                }
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < N; c += 16) tmem_st16(col + c, z);
                if (wrap_ok && slot >= (uint32_t)(NSLOT - 2)) {
                    // ring rows 0 / 1: the wrapped part of their sum sits in an extension slot
                    const uint32_t ecol = lane_base + (uint32_t)(2 * NSLOT - 1 - slot) * N;
#pragma unroll
                    for (int c = 0; c < N; c += 16) {
                        uint32_t t[16];
                        tmem_ld16(ecol + c, t);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            v[c + i] = __float_as_uint(__uint_as_float(v[c + i]) + __uint_as_float(t[i]));
                        tmem_st16(ecol + c, z);
                    }
                }
                tmem_wait_st();
                } else {
#pragma unroll
                    for (int i = 0; i < N; ++i) v[i] = 0u;
                }
                tc_fence_before();
                if constexpr (PAIR) {
                    __syncwarp();
                    if (lane == 0) {
                        if (rank == 0) mbar_arrive(&tempty[slot]);
                        else mbar_arrive_remote(lead_tempty + slot * 8);
                    }
                } else {
                    mbar_arrive(&tempty[slot]);
                }
                if (w < p.Wout && !(p.dbg & 1) && p.yf) {
                    // fp32 output (bf16x3 path): any channel stride, one value per channel
                    const int qo = q0 + j;
                    float *dst;
                    int64_t cs;
                    if (p.ysplit_dim == 0 && po >= p.ysplit) {
                        dst = p.yf2 + b * p.y2s[0] + (int64_t)(po - p.ysplit) * p.y2s[1] +
                              (int64_t)qo * p.y2s[2] + (int64_t)w * p.y2s[3];
                        cs = p.y2cs;
                    } else if (p.ysplit_dim == 1 && qo >= p.ysplit) {
                        dst = p.yf2 + b * p.y2s[0] + (int64_t)po * p.y2s[1] +
                              (int64_t)(qo - p.ysplit) * p.y2s[2] + (int64_t)w * p.y2s[3];
                        cs = p.y2cs;
                    } else {
                        dst = p.yf + b * p.ys[0] + (int64_t)po * p.ys[1] + (int64_t)qo * p.ys[2] +
                              (int64_t)w * p.ys[3];
                        cs = p.ycs;
                    }
#pragma unroll
                    for (int c = 0; c < N; ++c) dst[c * cs] = __uint_as_float(v[c]);
                } else if (w < p.Wout && !(p.dbg & 1)) {
                    const int qo = q0 + j;
                    __nv_bfloat16 *dst;
                    if (p.ysplit_dim == 0 && po >= p.ysplit)
                        dst = p.y2 + b * p.y2s[0] + (int64_t)(po - p.ysplit) * p.y2s[1] +
                              (int64_t)qo * p.y2s[2] + (int64_t)w * p.y2s[3];
                    else if (p.ysplit_dim == 1 && qo >= p.ysplit)
                        dst = p.y2 + b * p.y2s[0] + (int64_t)po * p.y2s[1] +
                              (int64_t)(qo - p.ysplit) * p.y2s[2] + (int64_t)w * p.y2s[3];
                    else
                        dst = p.y + b * p.ys[0] + (int64_t)po * p.ys[1] + (int64_t)qo * p.ys[2] +
                              (int64_t)w * p.ys[3];
#pragma unroll
                    for (int c = 0; c < N; c += 8) {
                        uint4 pk;
                        pk.x = pack_bf16(__uint_as_float(v[c + 0]), __uint_as_float(v[c + 1]));
                        pk.y = pack_bf16(__uint_as_float(v[c + 2]), __uint_as_float(v[c + 3]));
                        pk.z = pack_bf16(__uint_as_float(v[c + 4]), __uint_as_float(v[c + 5]));
                        pk.w = pack_bf16(__uint_as_float(v[c + 6]), __uint_as_float(v[c + 7]));
                        *reinterpret_cast<uint4 *>(dst + c) = pk;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        if constexpr (PAIR) tmem_dealloc2(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

// Output channel held by accumulator column `col` (0..N-1) when the bf16
// epilogue's coalesced 16x128b drain is used: column 4 j + c (c = col % 4, the
// lane-within-voxel of the fragment) carries channel U (4 (j / U) + c) + j % U,
// U = 8 (N % 32 == 0) or 4, so thread c of a voxel owns whole U-channel chunks.
__host__ __device__ __forceinline__ int epi_channel(int col, int N) {
    const int U = (N % 32 == 0) ? 8 : 4;
    const int j = col >> 2, c = col & 3;
    return U * (4 * (j / U) + c) + j % U;
}

// Weight smem image.  One block per (kp, kw, 16-channel kc) with KQ*N rows
// n = kq*N + c_out (the merged-tap MMA's B operand), UMMA K-major canonical:
// [n/8 group][k half][8 rows][8 k] bf16 -> SBO 256 B, LBO 128 B.
// flip=1 builds the dgrad weights W'[n=ci][k=co][t] = W[co][ci][taps-1-t].
__global__ void conv_tc_weight_image(const __nv_bfloat16 *__restrict__ w,
                                     __nv_bfloat16 *__restrict__ img, int n_rows, int k_cols,
                                     int KP, int KQ, int KW, int flip, int cperm) {
    const int KC = k_cols / 16;
    const int taps = KP * KQ * KW;
    const int NB = KQ * n_rows;  // rows per block
    const int total = KP * KW * KC * NB * 16;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        int r = e;
        const int kk = r % 8; r /= 8;
        const int nn = r % 8; r /= 8;
        const int h = r % 2; r /= 2;
        const int g = r % (NB / 8); r /= (NB / 8);
        const int kc = r % KC; r /= KC;
        const int kw = r % KW;
        const int kp = r / KW;
        const int nrow = g * 8 + nn;
        const int kq = nrow / n_rows;
        const int n = cperm ? epi_channel(nrow % n_rows, n_rows) : nrow % n_rows;
        const int k = kc * 16 + h * 8 + kk;
        const int t = (kp * KQ + kq) * KW + kw;
        __nv_bfloat16 v;
        if (!flip)
            v = w[((int64_t)n * k_cols + k) * taps + t];                  // W[co=n][ci=k][t]
        else
            v = w[((int64_t)k * n_rows + n) * taps + (taps - 1 - t)];    // W[co=k][ci=n][T-1-t]
        img[e] = v;
    }
}

// CTA-pair weight image: [rank][merged halves][per-kq halves].  Merged block
// (kp, kw, kc): rows n = r*KQ*N/2 + nn of the KQ*N merged rows (n = kq*N + c);
// per-kq block (kp, kw, kc, kq): rows c = r*N/2 + nn.  Canonical K-major as
// conv_tc_weight_image; flip = the dgrad image.
__global__ void conv_tc_weight_image_pair(const __nv_bfloat16 *__restrict__ w,
                                          __nv_bfloat16 *__restrict__ img, int n_rows, int k_cols,
                                          int KP, int KQ, int KW, int flip, int cperm) {
    const int KC = k_cols / 16;
    const int taps = KP * KQ * KW;
    const int MH = KQ * n_rows / 2, QH = n_rows / 2;          // rows per half block
    const int nblk = KP * KW * KC;
    const int per_cta = nblk * (MH + KQ * QH) * 16;           // elements
    const int total = 2 * per_cta;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int r = e / per_cta;
        int x = e % per_cta;
        int kq, c, bi, nn;
        int rows;
        if (x < nblk * MH * 16) {
            rows = MH;
            bi = x / (MH * 16);
            x %= MH * 16;
        } else {
            x -= nblk * MH * 16;
            rows = QH;
            const int bj = x / (QH * 16);
            x %= QH * 16;
            bi = bj / KQ;
            kq = bj % KQ;
        }
        const int kk = x % 8;
        const int nn8 = (x / 8) % 8;
        const int h = (x / 64) % 2;
        const int g = x / 128;
        nn = g * 8 + nn8;
        if (rows == MH) {
            const int n = r * MH + nn;
            kq = n / n_rows;
            c = n % n_rows;
        } else {
            c = r * QH + nn;
        }
        const int kc = bi % KC, kw = (bi / KC) % KW, kp = bi / (KC * KW);
        const int k = kc * 16 + h * 8 + kk;
        const int t = (kp * KQ + kq) * KW + kw;
        if (cperm) c = epi_channel(c, n_rows);
        img[e] = !flip ? w[((int64_t)c * k_cols + k) * taps + t]
                       : w[((int64_t)k * n_rows + c) * taps + (taps - 1 - t)];
    }
}

// Map a dp_conv_geom onto the (P, Q, W) roles.  Returns false if the
// configuration is outside this kernel's envelope.
struct Roles {
    int nsp;
    int Pin, Qin, Win, Pout, Qout, Wout;
    int KP, KQ, KW;
    int base_p, base_q, base_w;
    int split;
    int64_t xs[4], hs[4], ys[4];  // (b, p, q, w) element strides
};

bool map_roles(const dp_conv_geom *g, bool dgrad, Roles &R) {
    if (g->nsp != 2 && g->nsp != 3) return false;
    for (int i = 0; i < g->nsp; ++i)
        if (g->stride[i] != 1) return false;
    if (!(g->shard == -1 || g->shard == 0)) return false;
    R.nsp = g->nsp;
    // "input" of the kernel: x (fwd) or dy (dgrad); "output": y (fwd) or dx (dgrad)
    const int64_t *in_ext = dgrad ? g->out_ext : g->in_ext;
    const int64_t *out_ext = dgrad ? g->in_ext : g->out_ext;
    const int64_t *is = dgrad ? g->ys : g->xs;
    const int64_t *os = dgrad ? g->xs : g->ys;
    int k[3] = {g->kernel[0], g->kernel[1], g->kernel[2]};
    int64_t base[3];
    for (int i = 0; i < 3; ++i)
        base[i] = dgrad ? -(g->base[i] + k[i] - 1) : g->base[i];
    int64_t oext[3] = {out_ext[0], out_ext[1], out_ext[2]};
    if (dgrad && g->shard == 0) oext[0] += g->halo;  // virtual rows [0, in + halo)
    if (g->nsp == 3) {
        R.Pin = (int)in_ext[0]; R.Qin = (int)in_ext[1]; R.Win = (int)in_ext[2];
        R.Pout = (int)oext[0]; R.Qout = (int)oext[1]; R.Wout = (int)oext[2];
        R.KP = k[0]; R.KQ = k[1]; R.KW = k[2];
        R.base_p = (int)base[0]; R.base_q = (int)base[1]; R.base_w = (int)base[2];
        R.split = g->shard == 0 ? 0 : -1;
        for (int i = 0; i < 4; ++i) {
            int src = i == 0 ? 0 : i + 1;
            R.xs[i] = is[src];
            R.hs[i] = g->hs[src];
            R.ys[i] = os[src];
        }
    } else {
        R.Pin = 1; R.Qin = (int)in_ext[0]; R.Win = (int)in_ext[1];
        R.Pout = 1; R.Qout = (int)oext[0]; R.Wout = (int)oext[1];
        R.KP = 1; R.KQ = k[0]; R.KW = k[1];
        R.base_p = 0; R.base_q = (int)base[0]; R.base_w = (int)base[1];
        R.split = g->shard == 0 ? 1 : -1;
        R.xs[0] = is[0]; R.xs[1] = is[0]; R.xs[2] = is[2]; R.xs[3] = is[3];
        R.hs[0] = g->hs[0]; R.hs[1] = g->hs[0]; R.hs[2] = g->hs[2]; R.hs[3] = g->hs[3];
        R.ys[0] = os[0]; R.ys[1] = os[0]; R.ys[2] = os[2]; R.ys[3] = os[3];
    }
    return true;
}

int pick_n(int n) { return (n == 16 || n == 32 || n == 48 || n == 64 || n == 128) ? n : 0; }

struct Plan {
    Roles R;
    int Cin, N;           // K channels, N channels of this conv
    int cblk, stage_bytes, wimg_bytes, nstage, smem;
    bool x3;              // 6-block K over a 3-part activation (the bf16x3 path)
    int ppn;              // output planes per unit (2: P-pair, two TMEM rings)
};

bool make_plan(const dp_conv_geom *g, bool dgrad, Plan &pl, bool f32out = false, bool x3 = false,
               bool allow_pp = true) {
    if (!map_roles(g, dgrad, pl.R)) return false;
    pl.Cin = (int)(dgrad ? g->c_out : g->c_in);
    pl.N = pick_n((int)(dgrad ? g->c_in : g->c_out));
    if (!pl.N || pl.Cin % 16 || pl.Cin > 192) return false;
    if (pl.Cin > 128 && !(pl.R.KP == 1 && pl.R.KQ == 3 && pl.R.KW == 3)) return false;
    const Roles &R = pl.R;
    if (R.KW > 15 || R.KQ > 7 || R.KP > 7) return false;
    if (R.KQ * pl.N > 256) return false;                 // merged-tap MMA: N <= 256
    if (R.KQ + 2 > ring_slots(pl.N)) return false;       // TMEM ring
    // channel stride 1 on input and output, 16-B aligned row strides
    const int64_t *is = dgrad ? g->ys : g->xs;
    const int64_t *os = dgrad ? g->xs : g->ys;
    if (is[1] != 1 || (!f32out && os[1] != 1)) return false;
    // the halo block is an input in the forward (TMA: 16-B strides) and a bf16 /
    // fp32 output in dgrad
    if (g->halo > 0 && !(dgrad && f32out) && g->hs[1] != 1) return false;
    for (int i = 0; i < 4; ++i) {
        if (R.xs[i] % 8 || (!f32out && R.ys[i] % 8)) return false;
        if (g->halo > 0 && !(dgrad && f32out) && R.hs[i] % 8) return false;
    }
    if (x3 && !(R.KP == 1 && R.KQ == 3 && R.KW == 3 && (pl.Cin == 96 || pl.Cin == 192) &&
                (pl.N == 16 || pl.N == 32)))
        return false;
    pl.x3 = x3;
    pl.cblk = x3 ? pl.Cin / 6 : chan_block(pl.Cin);       // X3: one box per stored part
    // P-pair units for the hot 3-D shapes with a bf16 output: each input row then
    // crosses L2 -> SMEM twice per two planes instead of three times per plane
    static const bool pp_off = getenv("DP_CONV_PP") && getenv("DP_CONV_PP")[0] == '0';
    pl.ppn = (allow_pp && !pp_off && !x3 && !f32out && R.nsp == 3 && R.KP == 3 && R.KQ == 3 && R.KW == 3 &&
              (pl.Cin == 16 || pl.Cin == 32) && (pl.N == 16 || pl.N == 32) && R.Pout >= 2 &&
              R.KQ + 2 <= ring_slots(pl.N, 256)) ? 2 : 1;
    pl.stage_bytes = (R.KP + pl.ppn - 1) * (x3 ? 3 : pl.Cin / pl.cblk) * box_bytes(pl.cblk, R.KW);
    pl.wimg_bytes = R.KP * R.KQ * R.KW * pl.Cin * pl.N * 2;
    const int budget = 220 * 1024;
    const int fixed = ((pl.wimg_bytes + 1023) & ~1023) + 1024;
    int ns = (budget - fixed) / pl.stage_bytes;
    // measured: 4 stages suit the 27-KB stages of C_in = 32 (L2 fwd / dgrad
    // 0.755 -> 0.745 ms), the 15-KB C_in = 16 stages want 6-8
    const int ns_cap = pl.stage_bytes > 16384 ? 4 : 8;
    if (ns > ns_cap) ns = ns_cap;
    if (ns < 2) return false;
    pl.nstage = ns;
    pl.smem = fixed + ns * pl.stage_bytes;
    return true;
}

template <int N, int KP, int KQ, int KW, int CIN, bool X3 = false, int PPN = 1>
int launch_k(const CUtensorMap &xm, const CUtensorMap &hm, const ConvTcParams &p, int grid,
             int smem, cudaStream_t st) {
    auto kern = conv_tc_kernel<N, KP, KQ, KW, CIN, false, X3, PPN>;
    DP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, st>>>(xm, hm, p);
    return launch_status("conv_tc_kernel");
}

// CTA-pair instantiation: (2, 1, 1) clusters, grid = 2 x clusters
template <int N, int KP, int KQ, int KW, int CIN, bool X3 = false, int PPN = 1>
int launch_k_pair(const CUtensorMap &xm, const CUtensorMap &hm, const ConvTcParams &p, int grid,
                  int smem, cudaStream_t st) {
    auto kern = conv_tc_kernel<N, KP, KQ, KW, CIN, true, X3, PPN>;
    DP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, xm, hm, p));
    return launch_status("conv_tc_kernel<pair>");
}

// shapes with a CTA-pair instantiation (the hot, statically unrolled ones)
bool pair_shape(int N, int KP, int KQ, int KW, int Cin) {
    const bool k333 = KP == 3 && KQ == 3 && KW == 3, k133 = KP == 1 && KQ == 3 && KW == 3;
    static const bool p64_off = getenv("DP_CONV_PAIR64") && getenv("DP_CONV_PAIR64")[0] == '0';
    if (N == 64) return !p64_off && k133 && Cin == 64;   // cfg4's 2-D 64 -> 64 layers
    if (!(N == 16 || N == 32)) return false;
    return (k333 && (Cin == 16 || Cin == 32)) ||
           (k133 && (Cin == 32 || Cin == 64 || Cin == 96 || Cin == 192));
}

template <int N>
int launch_n_pair(const CUtensorMap &xm, const CUtensorMap &hm, const ConvTcParams &p, int grid,
                  int smem, cudaStream_t st) {
    const bool k333 = p.KP == 3 && p.KQ == 3 && p.KW == 3;
    if (k333 && p.Cin == 16) return launch_k_pair<N, 3, 3, 3, 16>(xm, hm, p, grid, smem, st);
    if (k333 && p.Cin == 32) return launch_k_pair<N, 3, 3, 3, 32>(xm, hm, p, grid, smem, st);
    if (p.Cin == 32) return launch_k_pair<N, 1, 3, 3, 32>(xm, hm, p, grid, smem, st);
    if (p.Cin == 64) return launch_k_pair<N, 1, 3, 3, 64>(xm, hm, p, grid, smem, st);
    if (p.Cin == 96) return launch_k_pair<N, 1, 3, 3, 96>(xm, hm, p, grid, smem, st);
    return launch_k_pair<N, 1, 3, 3, 192>(xm, hm, p, grid, smem, st);
}

// Hot shapes get a fully unrolled instantiation; everything else in the
// envelope runs the runtime-shaped kernel.
template <int N>
int launch_n(const CUtensorMap &xm, const CUtensorMap &hm, const ConvTcParams &p, int grid,
             int smem, cudaStream_t st) {
    const bool k333 = p.KP == 3 && p.KQ == 3 && p.KW == 3;
    const bool k133 = p.KP == 1 && p.KQ == 3 && p.KW == 3;
    if (k333 && p.Cin == 16) return launch_k<N, 3, 3, 3, 16>(xm, hm, p, grid, smem, st);
    if (k333 && p.Cin == 32) return launch_k<N, 3, 3, 3, 32>(xm, hm, p, grid, smem, st);
    if (k133 && p.Cin == 32) return launch_k<N, 1, 3, 3, 32>(xm, hm, p, grid, smem, st);
    if (k133 && p.Cin == 64) return launch_k<N, 1, 3, 3, 64>(xm, hm, p, grid, smem, st);
    if constexpr (N == 16 || N == 32) {     // the bf16x3 fp32 path: 6 x 16 / 6 x 32 channels
        if (k133 && p.Cin == 96) return launch_k<N, 1, 3, 3, 96>(xm, hm, p, grid, smem, st);
        if (k133 && p.Cin == 192) return launch_k<N, 1, 3, 3, 192>(xm, hm, p, grid, smem, st);
    }
    return launch_k<N, 0, 0, 0, 0>(xm, hm, p, grid, smem, st);
}

int run_conv_tc(const dp_conv_geom *g, bool dgrad, const void *in, const void *in_halo,
                const void *w, void *out, void *out2, void *ws, int64_t ws_bytes,
                cudaStream_t st, bool f32out = false, bool x3 = false) {
    Plan pl;
    DP_REQUIRE(make_plan(g, dgrad, pl, f32out, x3), DP_ERR_UNSUPPORTED,
               "conv_tc: outside the envelope");
    const Roles &R = pl.R;
    const int taps = R.KP * R.KQ * R.KW;
    DP_REQUIRE(ws_bytes >= pl.wimg_bytes, DP_ERR_INVALID, "conv_tc: workspace too small");
    int64_t outs = (int64_t)g->batch * R.Pout * R.Qout * R.Wout;
    if (outs == 0) return DP_OK;
    // CTA pairs (cta_group::2) over two adjacent W tiles when the shape has an
    // instantiation, there are >= 2 tiles and the workspace holds both images
    const int n_wt_all = (R.Wout + kTileW - 1) / kTileW;
    static const bool pair_off = getenv("DP_CONV_2CTA") && getenv("DP_CONV_2CTA")[0] == '0';
    const bool use_pair = !pair_off && n_wt_all >= 2 && sm_count() >= 2 &&
                          pair_shape(pl.N, R.KP, R.KQ, R.KW, pl.Cin) &&
                          ws_bytes >= 2 * (int64_t)pl.wimg_bytes;
    // bf16 outputs drain through the coalesced epilogue (permuted B columns) when
    // the halo output part shares the main part's W stride
    const bool split_out = dgrad && g->halo > 0 && g->shard == 0;
    const int cperm = (!f32out && (!split_out || R.hs[3] == R.ys[3])) ? 1 : 0;
    if (pl.ppn > 1 && !cperm)   // P-pair units drain through the coalesced epilogue only
        DP_REQUIRE(make_plan(g, dgrad, pl, f32out, x3, false), DP_ERR_UNSUPPORTED,
                   "conv_tc: outside the envelope");
    // weight image
    {
        int total = taps * pl.Cin * pl.N;
        if (use_pair)
            conv_tc_weight_image_pair<<<grid_for(2 * total, 256, 2), 256, 0, st>>>(
                (const __nv_bfloat16 *)w, (__nv_bfloat16 *)ws, pl.N, pl.Cin, R.KP, R.KQ, R.KW,
                dgrad ? 1 : 0, cperm);
        else
            conv_tc_weight_image<<<grid_for(total, 256, 2), 256, 0, st>>>(
                (const __nv_bfloat16 *)w, (__nv_bfloat16 *)ws, pl.N, pl.Cin, R.KP, R.KQ, R.KW,
                dgrad ? 1 : 0, cperm);
        int rc = launch_status("conv_tc_weight_image");
        if (rc) return rc;
    }
    // tensor maps: dims {C, W, Q, P, B}; box = one channel block x BW voxels
    const int BW = kTileW + R.KW - 1;
    uint32_t box[5] = {(uint32_t)pl.cblk, (uint32_t)BW, 1, 1, 1};
    const CUtensorMapSwizzle swz = pl.cblk == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                   : pl.cblk == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_128B;
    CUtensorMap xm, hm;
    {
        uint64_t dims[5] = {(uint64_t)(x3 ? pl.Cin / 6 : pl.Cin), (uint64_t)R.Win, (uint64_t)R.Qin,
                            (uint64_t)R.Pin, (uint64_t)(x3 ? 3 : 1) * g->batch};
        uint64_t strides[4] = {(uint64_t)R.xs[3] * 2, (uint64_t)R.xs[2] * 2,
                               (uint64_t)R.xs[1] * 2, (uint64_t)R.xs[0] * 2};
        int rc = encode_tensor_map(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(in),
                                   dims, strides, box, swz);
        if (rc) return rc;
    }
    hm = xm;
    if (!dgrad && g->halo > 0) {
        uint64_t dims[5] = {(uint64_t)(x3 ? pl.Cin / 6 : pl.Cin), (uint64_t)R.Win,
                            (uint64_t)(R.split == 1 ? g->halo : R.Qin),
                            (uint64_t)(R.split == 0 ? g->halo : R.Pin),
                            (uint64_t)(x3 ? 3 : 1) * g->batch};
        uint64_t strides[4] = {(uint64_t)R.hs[3] * 2, (uint64_t)R.hs[2] * 2,
                               (uint64_t)R.hs[1] * 2, (uint64_t)R.hs[0] * 2};
        int rc = encode_tensor_map(&hm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                                   const_cast<void *>(in_halo), dims, strides, box, swz);
        if (rc) return rc;
    }
    ConvTcParams p;
    memset(&p, 0, sizeof(p));
    p.B = (int)g->batch;
    p.Cin = pl.Cin;
    p.Cout = pl.N;
    p.Pin = R.Pin; p.Qin = R.Qin; p.Win = R.Win;
    p.Pout = R.Pout; p.Qout = R.Qout; p.Wout = R.Wout;
    p.KP = R.KP; p.KQ = R.KQ; p.KW = R.KW;
    p.base_p = R.base_p; p.base_q = R.base_q; p.base_w = R.base_w;
    p.split = dgrad ? -1 : (g->halo > 0 ? R.split : -1);
    p.halo = dgrad ? 0 : (int)g->halo;
    p.y = (__nv_bfloat16 *)out;
    p.y2 = (__nv_bfloat16 *)(out2 ? out2 : out);
    if (f32out) {
        p.yf = (float *)out;
        p.yf2 = (float *)(out2 ? out2 : out);
        p.ycs = dgrad ? g->xs[1] : g->ys[1];
        p.y2cs = g->hs[1];
    }
    for (int i = 0; i < 4; ++i) {
        p.ys[i] = R.ys[i];
        p.y2s[i] = R.hs[i];
    }
    p.cperm = cperm;
    p.ysplit_dim = -1;
    p.ysplit = 0;
    if (dgrad && g->halo > 0 && g->shard == 0) {
        p.ysplit_dim = R.split;                       // rows >= main extent -> dx_halo
        p.ysplit = R.split == 0 ? (int)g->in_ext[0] : (int)g->in_ext[0];
    }
    {
        const int64_t ns = ring_slots(pl.N, 512 / pl.ppn), q = g->nsp == 3 ? g->out_org[1] : g->out_org[0];
        p.qorg = (int)(((q % ns) + ns) % ns);
    }
    p.n_wt = use_pair ? (n_wt_all + 1) / 2 : n_wt_all;   // PAIR: tile pairs
    // choose the Q chunk so the unit count balances well over the SMs (pairs)
    const int sms = use_pair ? sm_count() / 2 : sm_count();
    p.Pu = (R.Pout + pl.ppn - 1) / pl.ppn;
    const int64_t cols = (int64_t)p.B * p.Pu * p.n_wt;
    int best_chunk = R.Qout;
    double best = -1;
    for (int nq = 1; nq <= R.Qout && nq <= 64; ++nq) {
        int chunk = (R.Qout + nq - 1) / nq;
        int nqc = (R.Qout + chunk - 1) / chunk;
        int64_t units = cols * nqc;
        int64_t waves = (units + sms - 1) / sms;
        double balance = (double)units / (double)(waves * sms);
        double overhead = (double)(chunk + R.KQ - 1) / chunk;
        double score = balance / overhead;
        if (score > best + 1e-9) {
            best = score;
            best_chunk = chunk;
        }
    }
    p.q_chunk = best_chunk;
    p.n_qc = (R.Qout + best_chunk - 1) / best_chunk;
    p.n_units = (int)(cols * p.n_qc);
    p.nstage = pl.nstage;
    p.wimg_bytes = pl.wimg_bytes;
    p.wimg = (const __nv_bfloat16 *)ws;
    {
        static int dbg = -1;
        if (dbg < 0) {
            const char *e = getenv("DP_CONV_DBG");
            dbg = e ? atoi(e) : 0;
        }
        p.dbg = dbg;
    }
    int grid = p.n_units < sms ? p.n_units : sms;
    if (pl.ppn == 2) {   // P-pair units (3-D 3x3x3, bf16 out, C 16 / 32)
        const bool c16 = pl.Cin == 16;
        if (use_pair) {
            if (pl.N == 16)
                return c16 ? launch_k_pair<16, 3, 3, 3, 16, false, 2>(xm, hm, p, 2 * grid, pl.smem, st)
                           : launch_k_pair<16, 3, 3, 3, 32, false, 2>(xm, hm, p, 2 * grid, pl.smem, st);
            return c16 ? launch_k_pair<32, 3, 3, 3, 16, false, 2>(xm, hm, p, 2 * grid, pl.smem, st)
                       : launch_k_pair<32, 3, 3, 3, 32, false, 2>(xm, hm, p, 2 * grid, pl.smem, st);
        }
        if (pl.N == 16)
            return c16 ? launch_k<16, 3, 3, 3, 16, false, 2>(xm, hm, p, grid, pl.smem, st)
                       : launch_k<16, 3, 3, 3, 32, false, 2>(xm, hm, p, grid, pl.smem, st);
        return c16 ? launch_k<32, 3, 3, 3, 16, false, 2>(xm, hm, p, grid, pl.smem, st)
                   : launch_k<32, 3, 3, 3, 32, false, 2>(xm, hm, p, grid, pl.smem, st);
    }
    if (pl.x3) {   // N (output channels) and K (6 x the contracted channels) vary independently
        const bool k96 = pl.Cin == 96;
        if (use_pair) {
            if (pl.N == 16)
                return k96 ? launch_k_pair<16, 1, 3, 3, 96, true>(xm, hm, p, 2 * grid, pl.smem, st)
                           : launch_k_pair<16, 1, 3, 3, 192, true>(xm, hm, p, 2 * grid, pl.smem, st);
            return k96 ? launch_k_pair<32, 1, 3, 3, 96, true>(xm, hm, p, 2 * grid, pl.smem, st)
                       : launch_k_pair<32, 1, 3, 3, 192, true>(xm, hm, p, 2 * grid, pl.smem, st);
        }
        if (pl.N == 16)
            return k96 ? launch_k<16, 1, 3, 3, 96, true>(xm, hm, p, grid, pl.smem, st)
                       : launch_k<16, 1, 3, 3, 192, true>(xm, hm, p, grid, pl.smem, st);
        return k96 ? launch_k<32, 1, 3, 3, 96, true>(xm, hm, p, grid, pl.smem, st)
                   : launch_k<32, 1, 3, 3, 192, true>(xm, hm, p, grid, pl.smem, st);
    }
    if (use_pair)
        return pl.N == 16 ? launch_n_pair<16>(xm, hm, p, 2 * grid, pl.smem, st)
               : pl.N == 32 ? launch_n_pair<32>(xm, hm, p, 2 * grid, pl.smem, st)
                            : launch_k_pair<64, 1, 3, 3, 64>(xm, hm, p, 2 * grid, pl.smem, st);
    switch (pl.N) {
        case 16: return launch_n<16>(xm, hm, p, grid, pl.smem, st);
        case 32: return launch_n<32>(xm, hm, p, grid, pl.smem, st);
        case 48: return launch_n<48>(xm, hm, p, grid, pl.smem, st);
        case 64: return launch_n<64>(xm, hm, p, grid, pl.smem, st);
        default: return launch_n<128>(xm, hm, p, grid, pl.smem, st);
    }
}

// ---------------------------------------------------------------------------


// ---------------------------------------------------------------------------
// Weight gradient:
//   dW[co][ci][kp][kq][kw] = sum_{b,po,qo,wo} dY[b,po,qo,wo,co] *
//                            X_virtual[b, base_p+po+kp, base_q+qo+kq, base_w+wo+kw, ci]
// Substituting w' = wo + kw: dW[..kw] = sum_w' X[base_w + w'] * dY[w' - kw].
//
// A unit is a column (b, po, w' tile) and a chunk of output rows [q0, q1); like
// the forward kernel it streams INPUT rows along Q.  Step s loads
//   * input row q = base_q + q0 + s: KP x (channel blocks) boxes of
//     16*kt w' voxels, swizzled, into the X ring, and
//   * (s < nq) dY row q0 + s as KW copies, each TMA-loaded at w' - kw (zero
//     outside [0, Wout)), into the dY ring.
// Once input row j + KQ - 1 has landed, output row j's whole contribution is
//   D[M = (kq, kp, ci)][N = (kw, co)] += X_{j..j+KQ-1}[K = w'] . dY_j[K = w']
// with the KQ consecutive X rows read as ONE operand: the X ring slots are
// contiguous and the first KQ-1 slots are mirrored after the last, so rows
// j..j+KQ-1 are always adjacent boxes (uniform LBO).  Both operands are
// MN-major straight out of the swizzled TMA boxes (K = w' runs down the
// rows).  M tiles cover (kq, kp, ci) 128 rows at a time — 144 rows in 2
// tiles for C_in = 16 (was 3 per-kq tiles of 48), 192 in 2 for the 2-D
// 64-channel case — rows past KQ*KP*Cin read the next boxes (garbage rows,
// never reduced into dW).  Each X row is loaded once per unit.  All units of
// a CTA accumulate into the same TMEM tiles; the per-CTA partials
// [cta][m][n] are summed into dW by a deterministic reduction.
struct WgradTcParams {
    int B, Cin, N;                   // N = Cout (dY channels)
    int Pin, Qin, Win, Pout, Qout, Wout;
    int KP, KQ, KW;
    int base_p, base_q, base_w;
    int split, halo;
    int n_wt, n_qc, q_chunk, n_units, n_mt, kt;  // kt = 16-voxel K steps per w' tile
    int nx, nd;                      // X ring slots (plus KQ-1 mirrors) / dY ring depth
    float *partial;                  // [grid][n_mt*128][KW*N]
    int sdy;                         // dY staged ONCE per row (see wlayout)
};

struct WLayout {
    int cbx, nbx, boxx;              // X channel block, blocks, box bytes
    int cbd, nbd, boxd;              // dY channel block, blocks, box bytes
    int xslot, dslot, tail;          // ring slot bytes, garbage tail after the mirrors
};

// sdy (single dY copy): the dY row is staged ONCE, as kt*16 + KW - 1 rows
// starting at w' = w0 - (KW - 1), instead of KW copies each shifted by -kw.
// The B operand N = (a, co), a = KW - 1 - kw, then reads MN swizzle atom a
// at row a of that box: atoms overlap, one row (LBO = cbd * 2 bytes) apart —
// the swizzle is a function of the absolute shared address (as for the
// forward kernel's kw-shifted A), so each atom reads the rows TMA wrote.
// Needs one channel block (cout <= 64) and a box of <= 256 rows.  Cuts the
// dY TMA bytes and shared-memory writes KW-fold (cfg4: 768 -> 256 KB per
// output row, which had pushed the kernel past the smem write + read budget).
__host__ __device__ inline WLayout wlayout(int cin, int cout, int KP, int KQ, int KW, int kt,
                                           int n_mt, int sdy = 0) {
    WLayout L;
    L.cbx = chan_block(cin);
    L.nbx = cin / L.cbx;
    L.boxx = (kt * 16 * L.cbx * 2 + 1023) / 1024 * 1024;
    L.cbd = chan_block(cout);
    L.nbd = cout / L.cbd;
    L.boxd = ((kt * 16 + (sdy ? KW - 1 : 0)) * L.cbd * 2 + 1023) / 1024 * 1024;
    L.xslot = KP * L.nbx * L.boxx;
    L.dslot = (sdy ? 1 : KW) * L.nbd * L.boxd;
    const int over = (n_mt * 128 / L.cbx - KQ * KP * L.nbx) * L.boxx;
    L.tail = over > 0 ? over : 0;
    return L;
}

template <int N, int KP_, int KQ_, int KW_, int CIN_>
__global__ void __launch_bounds__(kThreads, 1)
conv_wgrad_tc_kernel(const __grid_constant__ CUtensorMap xmap,
                     const __grid_constant__ CUtensorMap hmap,
                     const __grid_constant__ CUtensorMap dmap, const WgradTcParams p) {
    using namespace tc;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);   // warp-uniform for ptxas
    const int lane = threadIdx.x & 31;
    constexpr bool kStatic = KP_ > 0;
    const int KP = kStatic ? KP_ : p.KP;
    const int KQ = kStatic ? KQ_ : p.KQ;
    const int KW = kStatic ? KW_ : p.KW;
    const int CIN = kStatic ? CIN_ : p.Cin;
    const int NMT = (KQ * KP * CIN + 127) / 128;
    const WLayout L = wlayout(CIN, N, KP, KQ, KW, p.kt, NMT, p.sdy);
    const int NT = KW * N;  // MMA N
    const int NXM = p.nx + KQ - 1;   // physical X slots incl. mirrors
    uint8_t *xring = smem;
    uint8_t *dring = smem + (size_t)NXM * L.xslot + L.tail;
    uint64_t *bars = reinterpret_cast<uint64_t *>(dring + (size_t)p.nd * L.dslot);
    uint64_t *xfull = bars, *xempty = xfull + p.nx;
    uint64_t *dfull = xempty + p.nx, *dempty = dfull + p.nd, *done = dempty + p.nd;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(NMT * NT)) ncols <<= 1;
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < p.nx; ++i) {
                mbar_init(&xfull[i], 1);
                mbar_init(&xempty[i], 1);
            }
            for (int i = 0; i < p.nd; ++i) {
                mbar_init(&dfull[i], 1);
                mbar_init(&dempty[i], 1);
            }
            mbar_init(done, 1);
            mbar_fence_init();
            tma_prefetch(&xmap);
            tma_prefetch(&hmap);
            tma_prefetch(&dmap);
        }
        __syncwarp();
        tmem_alloc_ool(tmem_slot, ncols);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int WK = p.kt * 16;  // w' voxels per tile

    if (warp == 0) {
        // ===================== TMA producer (whole warp, elected issue) =====================
        uint32_t pxi = 0, pxph = 0, pdi = 0, pdph = 0;   // X / dY ring slots and phases
        const uint32_t xrow = (uint32_t)(KP * L.nbx * WK * L.cbx * 2);
        const uint32_t dbytes = p.sdy ? (uint32_t)((WK + KW - 1) * L.cbd * 2)
                                      : (uint32_t)(KW * L.nbd * WK * L.cbd * 2);
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            int r = u;
            const int wt = r % p.n_wt; r /= p.n_wt;
            const int qc = r % p.n_qc; r /= p.n_qc;
            const int po = r % p.Pout;
            const int b = r / p.Pout;
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int nq = q1 - q0, nrows = nq + KQ - 1;
            const int w0 = wt * WK;
            for (int s = 0; s < nrows; ++s) {
                {   // X: input row q = base_q + q0 + s, all kp (and its mirror slot)
                    const uint32_t idx = pxi, ph = pxph;
                    if (++pxi == (uint32_t)p.nx) { pxi = 0; pxph ^= 1u; }
                    const bool mirror = (int)idx < KQ - 1;
                    mbar_wait(&xempty[idx], ph ^ 1);
                    mbar_expect_tx_e(&xfull[idx], mirror ? 2 * xrow : xrow);
                    const int qv = p.base_q + q0 + s;
                    for (int kp = 0; kp < KP; ++kp) {
                        const int pv = p.base_p + po + kp;
                        const CUtensorMap *map = &xmap;
                        int pc = pv, qcrd = qv;
                        if (p.split == 0 && pv >= p.Pin && pv < p.Pin + p.halo) {
                            map = &hmap;
                            pc = pv - p.Pin;
                        } else if (p.split == 1 && qv >= p.Qin && qv < p.Qin + p.halo) {
                            map = &hmap;
                            qcrd = qv - p.Qin;
                        }
                        for (int cb = 0; cb < L.nbx; ++cb) {
                            const size_t off = (size_t)(kp * L.nbx + cb) * L.boxx;
                            tma_load_5d_e(xring + (size_t)idx * L.xslot + off, map, &xfull[idx],
                                          cb * L.cbx, p.base_w + w0, qcrd, pc, b);
                            if (mirror)
                                tma_load_5d_e(xring + (size_t)(p.nx + idx) * L.xslot + off, map,
                                              &xfull[idx], cb * L.cbx, p.base_w + w0, qcrd, pc, b);
                        }
                    }
                }
                if (s < nq) {  // dY row q0 + s, KW shifted copies
                    const uint32_t idx = pdi, ph = pdph;
                    if (++pdi == (uint32_t)p.nd) { pdi = 0; pdph ^= 1u; }
                    mbar_wait(&dempty[idx], ph ^ 1);
                    mbar_expect_tx_e(&dfull[idx], dbytes);
                    uint8_t *dst = dring + (size_t)idx * L.dslot;
                    if (p.sdy)
                        tma_load_5d_e(dst, &dmap, &dfull[idx], 0, w0 - (KW - 1), q0 + s, po, b);
                    else
                        for (int kw = 0; kw < KW; ++kw)
                            for (int cb = 0; cb < L.nbd; ++cb)
                                tma_load_5d_e(dst + (size_t)(kw * L.nbd + cb) * L.boxd, &dmap,
                                              &dfull[idx], cb * L.cbd, w0 - kw, q0 + s, po, b);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, elected issue) =====================
        const uint32_t idesc = idesc_bf16(128, NT, 1, 1);
        const uint64_t a0 = sdesc_mn(smem_u32(xring), L.boxx, 8 * L.cbx * 2, swz_layout(L.cbx));
        const uint64_t b0 = sdesc_mn(smem_u32(dring), p.sdy ? L.cbd * 2 : L.boxd, 8 * L.cbd * 2,
                                     swz_layout(L.cbd));
        const uint32_t astep = (16 * L.cbx * 2) >> 4;  // one K step = 16 w' rows
        const uint32_t bstep = (16 * L.cbd * 2) >> 4;
        // the static shapes' steps as constants (grouped issue below)
        constexpr uint32_t AS8 = (16 * chan_block(CIN_ > 0 ? CIN_ : 16) * 2) >> 4;
        constexpr uint32_t BS8 = (16 * chan_block(N) * 2) >> 4;
        const uint32_t mstep = (128 / L.cbx * L.boxx) >> 4;
        // X / dY ring slots and phases carried as counters (no integer division
        // per row); the K-step loop is unrolled to its 16-step maximum with an
        // early exit (a runtime-bounded MMA loop costs issue cycles per MMA)
        uint32_t xidx = 0, xph = 0, didx = 0, dph = 0;
        uint32_t fresh = (1u << NMT) - 1u;  // accumulators not yet written
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            int r = u / p.n_wt;
            const int qc = r % p.n_qc;
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int nq = q1 - q0, nrows = nq + KQ - 1;
            uint32_t xs = xidx;          // X ring slot of this unit's output row j (kq = 0)
            for (int s = 0; s < nrows; ++s) {
                const uint32_t cx = xidx, cxph = xph;
                if (++xidx == (uint32_t)p.nx) { xidx = 0; xph ^= 1u; }
                mbar_wait(&xfull[cx], cxph);
                const int j = s - (KQ - 1);   // output row complete with this input row
                if (j < 0) continue;
                const uint32_t cd = didx, cdph = dph;
                if (++didx == (uint32_t)p.nd) { didx = 0; dph ^= 1u; }
                mbar_wait(&dfull[cd], cdph);
                tc_fence_after();
                const uint64_t ax = a0 + ((xs * L.xslot) >> 4);
                const uint64_t bd = b0 + ((cd * L.dslot) >> 4);
#pragma unroll
                for (int mt = 0; mt < NMT; ++mt) {
                    const uint32_t d = tmem + (uint32_t)(mt * NT);
                    const uint32_t bit = 1u << mt;
                    uint32_t acc = (fresh & bit) ? 0u : 1u;
                    fresh &= ~bit;
                    if (kStatic && p.kt == 8 && astep == AS8 && bstep == BS8) {
                        // one elect for the tile's 8 K steps (static shapes, 128-w' tiles)
                        mma_bf16_x8<AS8, BS8>(d, ax + mt * mstep, bd, idesc, acc);
                        continue;
                    }
#pragma unroll
                    for (int ks = 0; ks < 16; ++ks) {
                        if (ks >= p.kt) break;
                        mma_bf16_e(d, ax + mt * mstep + ks * astep, bd + ks * bstep, idesc, acc);
                        acc = 1u;
                    }
                }
                mma_commit_e(&dempty[cd]);            // dY row j is done
                mma_commit_e(&xempty[xs]);            // input row j: its last tap (kq = 0)
                uint32_t xn = xs + 1 == (uint32_t)p.nx ? 0u : xs + 1;
                if (j == nq - 1)                      // unit end: rows j+1.. are never kq=0
                    for (int t = 1; t < KQ; ++t) {
                        mma_commit_e(&xempty[xn]);
                        xn = xn + 1 == (uint32_t)p.nx ? 0u : xn + 1;
                    }
                xs = xs + 1 == (uint32_t)p.nx ? 0u : xs + 1;
            }
        }
        mma_commit_e(done);
    } else {
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;
        mbar_wait(done, 0);
        tc_fence_after();
        for (int t = 0; t < NMT; ++t) {
            float *dst = p.partial + ((size_t)(blockIdx.x * NMT + t) * 128 + m) * NT;
            for (int c = 0; c < NT; c += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + t * NT + c, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4 *>(dst + c + i) =
                        make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                    __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, ncols);
    }
}

constexpr int kRedCols = 32, kRedGroups = 8;   // deterministic partial reductions

// dw[co][ci][kp][kq][kw] = sum_cta partial[cta][row][a*N + co], row = (kq*KP + kp)*Cin + ci,
// a = kw (a = KW-1-kw with the single dY copy).  Two-level fixed-order sum
// as wgrad_ts_reduce (32 columns x 8 CTA groups per block).
__global__ void __launch_bounds__(kRedCols * kRedGroups)
wgrad_tc_reduce(const float *__restrict__ part, float *__restrict__ dw, int ctas, int n_mt, int KP,
                int KQ, int KW, int Cin, int N, int sdy) {
    __shared__ double red[kRedGroups][kRedCols + 1];
    const int NT = KW * N;
    const int total = KQ * KP * Cin * NT;          // real rows, partial layout order (coalesced)
    const size_t per_cta = (size_t)n_mt * 128 * NT;
    const int lo = threadIdx.x % kRedCols, g = threadIdx.x / kRedCols;
    const int o = blockIdx.x * kRedCols + lo;
    double s = 0.0;
    if (o < total) {
        int c = g;
        for (; c + 3 * kRedGroups < ctas; c += 4 * kRedGroups) {
            const float a0 = part[(size_t)c * per_cta + o];
            const float a1 = part[(size_t)(c + kRedGroups) * per_cta + o];
            const float a2 = part[(size_t)(c + 2 * kRedGroups) * per_cta + o];
            const float a3 = part[(size_t)(c + 3 * kRedGroups) * per_cta + o];
            s += (double)a0;
            s += (double)a1;
            s += (double)a2;
            s += (double)a3;
        }
        for (; c < ctas; c += kRedGroups) s += (double)part[(size_t)c * per_cta + o];
    }
    red[g][lo] = s;
    __syncthreads();
    if (g == 0 && o < total) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < kRedGroups; ++k) t += red[k][lo];
        const int row = o / NT, col = o % NT;
        const int a = col / N, co = col % N;
        const int kw = sdy ? KW - 1 - a : a;
        const int ci = row % Cin, kqkp = row / Cin;
        const int kp = kqkp % KP, kq = kqkp / KP;
        dw[(((co * Cin + ci) * KP + kp) * KQ + kq) * KW + kw] = (float)t;
    }
}

struct WPlan {
    Roles R;
    int Cin, N, n_mt, kt, n_wt, nx, nd, smem, grid, q_chunk, n_qc;
    int sdy;
    WLayout L;
    int64_t n_units;
};

bool make_wplan(const dp_conv_geom *g, WPlan &pl) {
    if (!map_roles(g, false, pl.R)) return false;
    const Roles &R = pl.R;
    pl.Cin = (int)g->c_in;
    pl.N = pick_n((int)g->c_out);
    if (!pl.N || pl.Cin % 16 || 128 % chan_block(pl.Cin) || pl.Cin > 128) return false;
    if (R.KW * pl.N > 256) return false;
    if (g->xs[1] != 1 || g->ys[1] != 1) return false;
    if (g->halo > 0 && g->hs[1] != 1) return false;
    for (int i = 0; i < 4; ++i) {
        if (R.xs[i] % 8 || R.ys[i] % 8) return false;
        if (g->halo > 0 && R.hs[i] % 8) return false;
    }
    pl.n_mt = (R.KQ * R.KP * pl.Cin + 127) / 128;
    if (pl.n_mt * R.KW * pl.N > 512) return false;   // TMEM accumulators
    // w' tiles: K steps of 16 voxels, up to 16 steps (256-row boxes), balanced
    const int wr = R.Wout + R.KW - 1;
    const int steps = (wr + 15) / 16;
    const int tiles0 = (steps + 15) / 16;
    const int kt0 = (steps + tiles0 - 1) / tiles0;
    // smem: X ring (KQ+1..KQ+2 slots, + KQ-1 mirrors + garbage tail), dY ring
    const int budget = 220 * 1024 - 512;
    pl.kt = 0;
    static const bool sdy_off = getenv("DP_WGRAD_SDY") && getenv("DP_WGRAD_SDY")[0] == '0';
    for (int kt = kt0; kt >= 1 && !pl.kt; --kt) {
        // one staged dY copy when the channels are one block and the box fits
        pl.sdy = (!sdy_off && pl.N == chan_block(pl.N) && kt * 16 + R.KW - 1 <= 256) ? 1 : 0;
        const WLayout L = wlayout(pl.Cin, pl.N, R.KP, R.KQ, R.KW, kt, pl.n_mt, pl.sdy);
        for (int nx = R.KQ + 2; nx >= R.KQ + 1; --nx) {
            const int nd = 3;
            const int need = (nx + R.KQ - 1) * L.xslot + L.tail + nd * L.dslot;
            if (need <= budget) {
                pl.kt = kt;
                pl.L = L;
                pl.nx = nx;
                pl.nd = nd;
                break;
            }
        }
    }
    if (pl.kt < 1) return false;
    pl.n_wt = (steps + pl.kt - 1) / pl.kt;
    pl.smem = (pl.nx + R.KQ - 1) * pl.L.xslot + pl.L.tail + pl.nd * pl.L.dslot + 512;
    // q chunks: balance units over the SMs, amortise the KQ-1 extra rows
    const int sms = sm_count();
    const int64_t cols = (int64_t)g->batch * R.Pout * pl.n_wt;
    int best_chunk = R.Qout;
    double best = -1;
    for (int nq = 1; nq <= R.Qout && nq <= 64; ++nq) {
        const int chunk = (R.Qout + nq - 1) / nq;
        const int nqc = (R.Qout + chunk - 1) / chunk;
        const int64_t units = cols * nqc;
        const int64_t waves = (units + sms - 1) / sms;
        const double balance = (double)units / (double)(waves * sms);
        const double overhead = (double)(chunk + R.KQ - 1) / chunk;
        const double score = balance / overhead;
        if (score > best + 1e-9) {
            best = score;
            best_chunk = chunk;
        }
    }
    pl.q_chunk = best_chunk;
    pl.n_qc = (R.Qout + best_chunk - 1) / best_chunk;
    pl.n_units = cols * pl.n_qc;
    pl.grid = (int)(pl.n_units < sms ? pl.n_units : sms);
    if (pl.grid < 1) pl.grid = 1;
    return true;
}

template <int N, int KP, int KQ, int KW, int CIN>
int launch_wgrad_k(const CUtensorMap &xm, const CUtensorMap &hm, const CUtensorMap &dm,
                   const WgradTcParams &p, int grid, int smem, cudaStream_t st) {
    auto kern = conv_wgrad_tc_kernel<N, KP, KQ, KW, CIN>;
    DP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, st>>>(xm, hm, dm, p);
    return launch_status("conv_wgrad_tc_kernel");
}

template <int N>
int launch_wgrad_n(const CUtensorMap &xm, const CUtensorMap &hm, const CUtensorMap &dm,
                   const WgradTcParams &p, int grid, int smem, cudaStream_t st) {
    const bool k333 = p.KP == 3 && p.KQ == 3 && p.KW == 3;
    const bool k133 = p.KP == 1 && p.KQ == 3 && p.KW == 3;
    if (k333 && p.Cin == 16) return launch_wgrad_k<N, 3, 3, 3, 16>(xm, hm, dm, p, grid, smem, st);
    if (k333 && p.Cin == 32) return launch_wgrad_k<N, 3, 3, 3, 32>(xm, hm, dm, p, grid, smem, st);
    if (k133 && p.Cin == 64) return launch_wgrad_k<N, 1, 3, 3, 64>(xm, hm, dm, p, grid, smem, st);
    return launch_wgrad_k<N, 0, 0, 0, 0>(xm, hm, dm, p, grid, smem, st);
}

int run_wgrad_tc(const dp_conv_geom *g, const void *x, const void *xh, const void *dy, float *dw,
                 void *ws, int64_t ws_bytes, cudaStream_t st) {
    WPlan pl;
    DP_REQUIRE(make_wplan(g, pl), DP_ERR_UNSUPPORTED, "conv_wgrad_tc: outside the envelope");
    const Roles &R = pl.R;
    const int64_t need = (int64_t)pl.grid * pl.n_mt * 128 * R.KW * pl.N * 4;
    DP_REQUIRE(ws_bytes >= need, DP_ERR_INVALID, "conv_wgrad_tc: workspace too small");
    (void)need;
    const int taps = R.KP * R.KQ * R.KW;
    if (pl.n_units == 0) {
        DP_CUDA_CHECK(cudaMemsetAsync(dw, 0, (size_t)pl.N * pl.Cin * taps * 4, st));
        return DP_OK;
    }
    const WLayout &L = pl.L;
    const uint32_t wk = (uint32_t)pl.kt * 16;
    auto swz = [](int cb) {
        return cb == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                        : cb == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    };
    uint32_t xbox[5] = {(uint32_t)L.cbx, wk, 1, 1, 1};
    CUtensorMap xm, hm, dm;
    {
        uint64_t dims[5] = {(uint64_t)pl.Cin, (uint64_t)R.Win, (uint64_t)R.Qin, (uint64_t)R.Pin,
                            (uint64_t)g->batch};
        uint64_t strides[4] = {(uint64_t)R.xs[3] * 2, (uint64_t)R.xs[2] * 2,
                               (uint64_t)R.xs[1] * 2, (uint64_t)R.xs[0] * 2};
        int rc = encode_tensor_map(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(x),
                                   dims, strides, xbox, swz(L.cbx));
        if (rc) return rc;
    }
    hm = xm;
    if (g->halo > 0) {
        uint64_t dims[5] = {(uint64_t)pl.Cin, (uint64_t)R.Win,
                            (uint64_t)(R.split == 1 ? g->halo : R.Qin),
                            (uint64_t)(R.split == 0 ? g->halo : R.Pin), (uint64_t)g->batch};
        uint64_t strides[4] = {(uint64_t)R.hs[3] * 2, (uint64_t)R.hs[2] * 2,
                               (uint64_t)R.hs[1] * 2, (uint64_t)R.hs[0] * 2};
        int rc = encode_tensor_map(&hm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                                   const_cast<void *>(xh), dims, strides, xbox, swz(L.cbx));
        if (rc) return rc;
    }
    {
        uint64_t dims[5] = {(uint64_t)pl.N, (uint64_t)R.Wout, (uint64_t)R.Qout, (uint64_t)R.Pout,
                            (uint64_t)g->batch};
        uint64_t strides[4] = {(uint64_t)R.ys[3] * 2, (uint64_t)R.ys[2] * 2,
                               (uint64_t)R.ys[1] * 2, (uint64_t)R.ys[0] * 2};
        uint32_t dbox[5] = {(uint32_t)L.cbd, wk + (pl.sdy ? (uint32_t)R.KW - 1 : 0u), 1, 1, 1};
        int rc = encode_tensor_map(&dm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(dy),
                                   dims, strides, dbox, swz(L.cbd));
        if (rc) return rc;
    }
    WgradTcParams p;
    memset(&p, 0, sizeof(p));
    p.B = (int)g->batch; p.Cin = pl.Cin; p.N = pl.N;
    p.Pin = R.Pin; p.Qin = R.Qin; p.Win = R.Win;
    p.Pout = R.Pout; p.Qout = R.Qout; p.Wout = R.Wout;
    p.KP = R.KP; p.KQ = R.KQ; p.KW = R.KW;
    p.base_p = R.base_p; p.base_q = R.base_q; p.base_w = R.base_w;
    p.split = g->halo > 0 ? R.split : -1;
    p.halo = (int)g->halo;
    p.n_wt = pl.n_wt; p.n_qc = pl.n_qc; p.q_chunk = pl.q_chunk;
    p.n_units = (int)pl.n_units;
    p.n_mt = pl.n_mt; p.kt = pl.kt;
    p.nx = pl.nx; p.nd = pl.nd;
    p.partial = (float *)ws;
    p.sdy = pl.sdy;
    int rc;
    switch (pl.N) {
        case 16: rc = launch_wgrad_n<16>(xm, hm, dm, p, pl.grid, pl.smem, st); break;
        case 32: rc = launch_wgrad_n<32>(xm, hm, dm, p, pl.grid, pl.smem, st); break;
        case 48: rc = launch_wgrad_n<48>(xm, hm, dm, p, pl.grid, pl.smem, st); break;
        default: rc = launch_wgrad_n<64>(xm, hm, dm, p, pl.grid, pl.smem, st); break;
    }
    if (rc) return rc;
    const int total = pl.N * pl.Cin * taps;
    wgrad_tc_reduce<<<(unsigned)((total + kRedCols - 1) / kRedCols), kRedCols * kRedGroups, 0, st>>>(
        (const float *)ws, dw, pl.grid, pl.n_mt, R.KP, R.KQ, R.KW, pl.Cin, pl.N, pl.sdy);
    return launch_status("wgrad_tc_reduce");
}


// ---------------------------------------------------------------------------
// Weight gradient, TS form (C_out = 32, KQ = KW = 3): dY in TMEM, X from smem.
//
//   D[m = (kw, co)][n = (kq, kp, ci)] += sum_w' dY[j][w' - kw][co] * X[j + kq][kp][w'][ci]
//
// The swapped roles put the 96 (kw, co) rows of one dY row into the A operand
// and ALL of the (kq, kp, ci) columns (144 / 192 / 288) into N, so every X
// row is read from shared memory exactly once per output row as a B operand
// (no per-M-tile re-reads) and the MMA runs at its N/2-cycle compute floor
// instead of the ~56-cycle shared-memory floor of the SS N = 96 form.  The A
// operand is built in TMEM by the 3 "transposer" warps (warp kw owns TMEM
// lanes 32 kw .. 32 kw + 31): per K = 16 step an ldmatrix.x4.trans of the
// staged dY row (rows w' - kw, re-ordered {0,1,4,5,..} / {2,3,6,7,..} so the
// transposed fragment IS the tcgen05 16x256b fragment) and one
// tcgen05.st.16x256b.  Lanes 96..127 are junk rows (never reduced).
// X rows come through a TMA ring like the SS kernel's (the KQ rows j..j+2 of
// output row j are adjacent slots, one uniform-LBO operand; a row whose KQ
// slots wrap past the ring end issues its B as two MMAs — no mirrored slots).
// Only the w' range where X is real is visited (the zero padding columns
// contribute nothing), so 256-wide rows are exactly two 128-voxel tiles.
constexpr int kTsCo = 32, kTsKT = 8, kTsWK = kTsKT * 16;
constexpr int kTsDRow = 16 * 2;                                  // staged dY half row: 16 co
constexpr int kTsDHalf = ((kTsWK + 2) * kTsDRow + 1023) / 1024 * 1024;  // one co half, 130 rows
constexpr int kTsDSlot = 2 * kTsDHalf;

struct WgradTsParams {
    int Pin, Qin, Win, Pout, Qout, Wout;
    int base_p, base_q, base_w;
    int split, halo;
    int w_lo, n_wt, n_qc, q_chunk, n_units;
    int nx, nd, na;
    float *partial;   // [grid][96][NT]
    int dbg;          // ablations (DP_CONV_DBG): 1 no transpose, 2 no MMA, 4 no TMA
    int rf_shift;     // RF: 2^rf_shift output rows per fresh D tile (flush group)
    int pairB;        // > 0: batch b = k * pairB + bb pairs X part kTsPairX[k] with dY part
                      // kTsPairD[k] (the bf16x3 fp32 wgrad: 6 pairings of 3 + 3 parts)
};
// part (hi 0, mid 1, lo 2) pairings of the bf16x3 wgrad, 2 bits per pairing k:
// X {0,1,0,2,1,0}, dY {0,0,1,0,1,2}
constexpr uint32_t kTsPairX = 0u | (1u << 2) | (0u << 4) | (2u << 6) | (1u << 8) | (0u << 10);
constexpr uint32_t kTsPairD = 0u | (0u << 2) | (1u << 4) | (0u << 6) | (1u << 8) | (2u << 10);

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
// 16 lanes x 16 repetitions of 128 bits: 64 consecutive columns (8 K = 16 steps);
// register 2j + g -> lane (lane_id / 4 + 8 g), column 4 j + lane_id % 4.
__device__ __forceinline__ void tmem_st_16x128b_x16(uint32_t addr, const uint32_t (&r)[8][4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x128b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};" ::"r"(addr),
        "r"(r[0][0]), "r"(r[0][1]), "r"(r[0][2]), "r"(r[0][3]), "r"(r[1][0]), "r"(r[1][1]),
        "r"(r[1][2]), "r"(r[1][3]), "r"(r[2][0]), "r"(r[2][1]), "r"(r[2][2]), "r"(r[2][3]),
        "r"(r[3][0]), "r"(r[3][1]), "r"(r[3][2]), "r"(r[3][3]), "r"(r[4][0]), "r"(r[4][1]),
        "r"(r[4][2]), "r"(r[4][3]), "r"(r[5][0]), "r"(r[5][1]), "r"(r[5][2]), "r"(r[5][3]),
        "r"(r[6][0]), "r"(r[6][1]), "r"(r[6][2]), "r"(r[6][3]), "r"(r[7][0]), "r"(r[7][1]),
        "r"(r[7][2]), "r"(r[7][3])
        : "memory");
}

template <int CIN, int KP>
struct TsShape {
    static constexpr int KQ = 3, KW = 3;
    static constexpr int CBX = chan_block(CIN);
    static constexpr int NBX = CIN / CBX;
    static constexpr int NATOM = KQ * KP * NBX;
    static constexpr int NT = NATOM * CBX;                 // MMA N total = KQ*KP*CIN
    static constexpr int NCH = (NT + 255) / 256;           // MMAs per K step
    static constexpr int APC = (NATOM + NCH - 1) / NCH;    // atoms per MMA (last may be short)
    static constexpr int BOXX = kTsWK * CBX * 2;           // one (kp, cb) X box
    static constexpr int XSLOT = KP * NBX * BOXX;
    static constexpr int ACOL = (NT + 31) / 32 * 32;       // first A column in TMEM
    static constexpr int ACOLS = kTsKT * 8;                // TMEM columns per A slot
    static_assert(BOXX % 1024 == 0, "X boxes must keep the swizzle atom alignment");
};

// RF (row flush, the bf16x3 fp32 wgrad): the tensor core adds into its fp32
// accumulator without round-to-nearest, and over a CTA's whole share of a
// 1M-voxel reduction that bias reached 2.6e-5 of max|dW| on cfg1 (above the
// reference's 1e-5).  With RF every output row accumulates into its own
// fresh TMEM tile (double-buffered D), and the transposer warps add it into
// per-thread fp32 registers (round-to-nearest FADD) right after staging the
// next row's A: the tensor-core chain is one row (8 K steps), the register
// chain the CTA's rows.
//
// G3 (the 2-D bf16x3 fp32 wgrad, grouped): a unit runs ALL 6 part pairings
// of its rows — an X ring slot holds the 3 X part boxes of a row, each dY part
// is staged and transposed ONCE per row (3 A entries), and the MMA warp issues
// the 6 pairings' K steps into the same D tile (every pairing adds into the
// same dW columns; each MMA's B spans one X part's KQ rows at the slot stride).
// Half the transposes and TMA bytes of running the pairings as batch entries.
template <int CIN, int KP, bool RF = false, bool G3 = false>
__global__ void __launch_bounds__(kThreads, 1)
conv_wgrad_ts_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
                     const __grid_constant__ CUtensorMap dmap, const WgradTsParams p) {
    using namespace tc;
    using S = TsShape<CIN, KP>;
    constexpr int KQ = S::KQ, KW = S::KW;
    constexpr int ACOL = RF ? (2 * S::NT + 31) / 32 * 32 : S::ACOL;   // first A column
    static_assert(!RF || S::NT <= 96, "row-flush registers: NT <= 96");
    static_assert(!G3 || (KP == 1 && RF), "G3: the 2-D bf16x3 wgrad");
    constexpr int NXP = G3 ? 3 : 1;            // X / dY parts per row (G3)
    constexpr int XS = NXP * S::XSLOT;         // X ring slot bytes
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);   // warp-uniform for ptxas
    const int lane = threadIdx.x & 31;
    // X ring: nx slots, no mirrored copies — an output row whose KQ input rows
    // wrap past the last slot issues its B operand as two MMAs (before / after
    // the wrap) instead of reading mirrored slots (those cost 2 / nx extra X
    // loads: 40 % of the X stream for the L2 shape's 5-slot ring)
    const int NXM = p.nx;
    uint8_t *xring = smem;
    uint8_t *dring = smem + (size_t)NXM * XS;
    uint64_t *bars = reinterpret_cast<uint64_t *>(dring + (size_t)p.nd * kTsDSlot);
    uint64_t *xfull = bars, *xempty = xfull + p.nx;
    uint64_t *dfull = xempty + p.nx, *dempty = dfull + p.nd;
    uint64_t *afull = dempty + p.nd, *aempty = afull + p.na, *done = aempty + p.na;
    uint64_t *rfull = done + 1, *rempty = rfull + 2;              // RF: D tile hand-off
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rempty + 2);
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < p.nx; ++i) {
                mbar_init(&xfull[i], 1);
                mbar_init(&xempty[i], 1);
            }
            for (int i = 0; i < p.nd; ++i) {
                mbar_init(&dfull[i], 1);
                mbar_init(&dempty[i], KW);
            }
            for (int i = 0; i < p.na; ++i) {
                mbar_init(&afull[i], KW);
                mbar_init(&aempty[i], 1);
            }
            mbar_init(done, 1);
            for (int i = 0; i < 2; ++i) {
                mbar_init(&rfull[i], 1);
                mbar_init(&rempty[i], KW);
            }
            mbar_fence_init();
            tma_prefetch(&xmap);
            tma_prefetch(&hmap);
            tma_prefetch(&dmap);
        }
        __syncwarp();
        tmem_alloc_ool(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        uint32_t pxi = 0, pxph = 0, pdi = 0, pdph = 0;   // X / dY ring slots and phases
        constexpr uint32_t xrow = (uint32_t)(KP * S::NBX * kTsWK * S::CBX * 2);
        constexpr uint32_t dbytes = 2u * (kTsWK + KW - 1) * kTsDRow;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            int r = u;
            const int wt = r % p.n_wt; r /= p.n_wt;
            const int qc = r % p.n_qc; r /= p.n_qc;
            const int po = r % p.Pout;
            const int b = r / p.Pout;
            int bx = b, bd = b;
            if (p.pairB > 0 && !G3) {
                const int kk = b / p.pairB, bb = b % p.pairB;
                bx = (int)((kTsPairX >> (2 * kk)) & 3u) * p.pairB + bb;
                bd = (int)((kTsPairD >> (2 * kk)) & 3u) * p.pairB + bb;
            }
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int nq = q1 - q0, nrows = nq + KQ - 1;
            const int w0 = p.w_lo + wt * kTsWK;
            for (int s = 0; s < nrows; ++s) {
                {
                    const uint32_t idx = pxi, ph = pxph;
                    if (++pxi == (uint32_t)p.nx) { pxi = 0; pxph ^= 1u; }
                    mbar_wait(&xempty[idx], ph ^ 1);
                    if (p.dbg & 4) {
                        if (lane == 0) mbar_arrive(&xfull[idx]);
                        __syncwarp();
                    } else {
                    mbar_expect_tx_e(&xfull[idx], xrow * NXP);
                    const int qv = p.base_q + q0 + s;
#pragma unroll
                    for (int kp = 0; kp < KP; ++kp) {
                        const int pv = p.base_p + po + kp;
                        const CUtensorMap *map = &xmap;
                        int pc = pv, qcrd = qv;
                        if (p.split == 0 && pv >= p.Pin && pv < p.Pin + p.halo) {
                            map = &hmap;
                            pc = pv - p.Pin;
                        } else if (p.split == 1 && qv >= p.Qin && qv < p.Qin + p.halo) {
                            map = &hmap;
                            qcrd = qv - p.Qin;
                        }
#pragma unroll
                        for (int xp = 0; xp < NXP; ++xp)
#pragma unroll
                        for (int cb = 0; cb < S::NBX; ++cb) {
                            const size_t off = (size_t)xp * S::XSLOT + (size_t)(kp * S::NBX + cb) * S::BOXX;
                            tma_load_5d_e(xring + (size_t)idx * XS + off, map, &xfull[idx],
                                          cb * S::CBX, p.base_w + w0, qcrd, pc,
                                          G3 ? xp * p.pairB + b : bx);
                        }
                    }
                    }
                }
                if (s < nq) {  // dY row q0 + s: two 16-channel halves, w' in [w0 - 2, w0 + 128)
                    for (int dp = 0; dp < NXP; ++dp) {   // G3: the 3 dY parts, one ring entry each
                    const uint32_t idx = pdi, ph = pdph;
                    if (++pdi == (uint32_t)p.nd) { pdi = 0; pdph ^= 1u; }
                    mbar_wait(&dempty[idx], ph ^ 1);
                    if (p.dbg & 4) {
                        if (lane == 0) mbar_arrive(&dfull[idx]);
                        __syncwarp();
                        continue;
                    }
                    mbar_expect_tx_e(&dfull[idx], dbytes);
                    uint8_t *dst = dring + (size_t)idx * kTsDSlot;
                    // G3: parts in the order the MMA warp first reads them (lo, mid, hi)
                    const int bdp = G3 ? (NXP - 1 - dp) * p.pairB + b : bd;
                    tma_load_5d_e(dst, &dmap, &dfull[idx], 0, w0 - (KW - 1), q0 + s, po, bdp);
                    tma_load_5d_e(dst + kTsDHalf, &dmap, &dfull[idx], 16, w0 - (KW - 1), q0 + s, po, bdp);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        // B atoms: (kq, kp, cb) boxes at one stride (G3: one X part's KQ rows, slot stride)
        const uint64_t b0 = sdesc_mn(smem_u32(xring), G3 ? XS : S::BOXX, 8 * S::CBX * 2,
                                     swz_layout(S::CBX));
        constexpr uint32_t bstep = (16 * S::CBX * 2) >> 4;   // one K step = 16 w' rows
        // ring slots / phases carried as counters (no integer division per row:
        // it costs MMA-warp issue time, cf. the fwd kernel)
        uint32_t xidx = 0, xph = 0, aidx = 0, aph = 0, rrow = 0;
        bool fresh = true;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            int r = u / p.n_wt;
            const int qc = r % p.n_qc;
            const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
            const int nq = q1 - q0, nrows = nq + KQ - 1;
            uint32_t xs = xidx;                    // X slot of output row j (= unit row j)
            for (int s = 0; s < nrows; ++s) {
                const uint32_t cx = xidx, cph = xph;
                if (++xidx == (uint32_t)p.nx) { xidx = 0; xph ^= 1u; }
                mbar_wait(&xfull[cx], cph);
                const int j = s - (KQ - 1);
                if (j < 0) continue;
                // this row's A entries (G3: one per dY part, staged lo, mid, hi — the
                // order the pairings first read them — each waited for just before its
                // first pairing and released after its last, so with 5 entries for 3
                // parts a row's first MMAs never wait for the previous row to finish)
                uint32_t cas[NXP], caph[NXP];
#pragma unroll
                for (int i = 0; i < NXP; ++i) {
                    const int dpi = G3 ? NXP - 1 - i : i;
                    cas[dpi] = aidx;
                    caph[dpi] = aph;
                    if (!G3) mbar_wait(&afull[aidx], aph);
                    if (++aidx == (uint32_t)p.na) { aidx = 0; aph ^= 1u; }
                }
                const uint32_t ca = cas[0];
                uint32_t dcol = tmem;
                if constexpr (RF) {   // group g = rrow / rf_rows uses D tile g & 1; a new
                                      // group's tile must have been drained (group g - 2)
                    const uint32_t g = (rrow >> p.rf_shift);
                    const uint32_t rb = g & 1u;
                    if ((rrow & ((1u << p.rf_shift) - 1u)) == 0) {
                        mbar_wait(&rempty[rb], ((g >> 1) & 1u) ^ 1u);
                        fresh = true;
                    }
                    dcol += rb * S::NT;
                }
                tc_fence_after();
                const uint64_t bx = b0 + ((xs * XS) >> 4);
                const uint32_t acol = tmem + ACOL + ca * S::ACOLS;
                if constexpr (G3) {
                    // the 6 pairings (X part kTsPairX[k], dY part kTsPairD[k]) into one D
                    const bool wrap = xs + KQ - 1 >= (uint32_t)p.nx;
                    const int aw = wrap ? (int)(p.nx - xs) : KQ;
                    const uint32_t id1 = idesc_bf16(128, aw * S::CBX, 0, 1);
                    const uint32_t id2 = idesc_bf16(128, (KQ - aw) * S::CBX, 0, 1);
                    // smallest products first (lo / mid pairings, then hi x hi): the tensor
                    // core's accumulator adds truncate, so the small terms go in while the
                    // tile's running sum is still small
#pragma unroll
                    for (int k = 5; k >= 0; --k) {
                        const uint32_t xp = (kTsPairX >> (2 * k)) & 3u, dp = (kTsPairD >> (2 * k)) & 3u;
                        const uint32_t ak = tmem + ACOL + cas[dp] * S::ACOLS;
                        const uint64_t bk = bx + ((xp * S::XSLOT) >> 4);
                        const uint64_t bk0 = b0 + ((xp * S::XSLOT) >> 4);
                        // the pairing's 8 K steps under one elect; a row whose KQ slots wrap
                        // the ring (2 of every nx rows) as two such groups over disjoint D
                        // columns (slots xs .. nx-1, then 0 ..)
                        static_assert(kTsKT == 8, "mma_ts_x8 covers one 128-w' tile");
                        if (k == 5 || k == 4 || k == 3) {   // first read of dY part dp
                            mbar_wait(&afull[cas[dp]], caph[dp]);
                            tc_fence_after();
                        }
                        if (!(p.dbg & 2)) {
                            const uint32_t acc0 = (fresh && k == 5) ? 0u : 1u;
                            mma_ts_x8<bstep>(dcol, ak, bk, id1, acc0);
                            if (wrap) mma_ts_x8<bstep>(dcol + aw * S::CBX, ak, bk0, id2, acc0);
                        }
                        if (k == 5 || k == 2 || k == 0)     // last read of dY part dp
                            mma_commit_e(&aempty[cas[dp]]);
                    }
                } else if (xs + KQ - 1 < (uint32_t)p.nx) {   // the KQ rows are adjacent slots
                    // per N chunk, its 8 K steps under one elect (the chunks write disjoint
                    // D columns, so chunk-outer order gives the same sums)
                    static_assert(kTsKT == 8, "mma_ts_x8 covers one 128-w' tile");
#pragma unroll
                    for (int c = 0; c < S::NCH; ++c) {
                        if (p.dbg & 2) break;
                        constexpr int last = S::NATOM - (S::NCH - 1) * S::APC;
                        const int atoms = c < S::NCH - 1 ? S::APC : last;
                        mma_ts_x8<bstep>(dcol + c * S::APC * S::CBX, acol,
                                         bx + ((c * S::APC * S::BOXX) >> 4),
                                         idesc_bf16(128, atoms * S::CBX, 0, 1), fresh ? 0u : 1u);
                    }
                } else {   // wrap: atoms of slots xs .. nx-1, then of slots 0 ..
                    const int aw = (int)(p.nx - xs) * KP * S::NBX;
                    const uint32_t id1 = idesc_bf16(128, aw * S::CBX, 0, 1);
                    const uint32_t id2 = idesc_bf16(128, (S::NATOM - aw) * S::CBX, 0, 1);
#pragma unroll
                    for (int ks = 0; ks < kTsKT; ++ks) {   // (grouped issue measured 0.7 % slower here)
                        if (p.dbg & 2) break;
                        const uint32_t acc = (fresh && ks == 0) ? 0u : 1u;
                        mma_ts_e(dcol, acol + ks * 8, bx + ks * bstep, id1, acc);
                        mma_ts_e(dcol + aw * S::CBX, acol + ks * 8, b0 + ks * bstep, id2, acc);
                    }
                }
                fresh = false;
                if constexpr (RF) {
                    if ((rrow & ((1u << p.rf_shift) - 1u)) == (1u << p.rf_shift) - 1u)
                        mma_commit_e(&rfull[((rrow >> p.rf_shift)) & 1u]);
                    ++rrow;
                }
                if constexpr (!G3) mma_commit_e(&aempty[cas[0]]);   // (G3: released per part)
                mma_commit_e(&xempty[xs]);
                uint32_t xn = xs + 1 == (uint32_t)p.nx ? 0u : xs + 1;
                if (j == nq - 1)
                    for (int t = 1; t < KQ; ++t) {
                        mma_commit_e(&xempty[xn]);
                        xn = xn + 1 == (uint32_t)p.nx ? 0u : xn + 1;
                    }
                xs = xs + 1 == (uint32_t)p.nx ? 0u : xs + 1;
            }
        }
        if constexpr (RF) {   // a last, partial flush group
            if ((rrow & ((1u << p.rf_shift) - 1u)) != 0)
                mma_commit_e(&rfull[(((rrow - 1) >> p.rf_shift)) & 1u]);
        }
        mma_commit_e(done);
    } else {
        // ===================== transposers (dY -> TMEM A), then epilogue =====================
        const int quarter = warp & 3;
        if (quarter < KW) {
            const int kw = quarter;
            // ldmatrix.x4.trans per K = 16 step: matrix mi = lane / 8 covers channels
            // 8 (mi & 1) .. +7 of the co half and w' rows 8 (mi >> 1) .. +7 (shifted by
            // -kw); row ri = lane % 8.  The staged half rows are 32 B with the TMA
            // 32-B swizzle (16-B chunk ^= row bit 2), so each matrix's 8 rows hit 8
            // distinct bank groups.  Transposed, thread t gets (co = t/4 [+8],
            // w' pair t%4 [+4]) = the 16x128b fragment, in x16 register order.
            const int mi = lane >> 3, ri = lane & 7;
            const int chunk = mi & 1;
            const int rbase = 8 * (mi >> 1) + ri + KW - 1 - kw;
            uint32_t didx = 0, dph = 0, aidx = 0, aph = 0, rrow = 0;
            float racc[RF ? S::NT : 1];
#pragma unroll
            for (int i = 0; i < (RF ? S::NT : 1); ++i) racc[i] = 0.f;
            // RF: add flush group g's D tile (this warp's lane quarter) into racc
            auto drain = [&](uint32_t g) {
                const uint32_t rb = g & 1u;
                mbar_wait(&rfull[rb], (g >> 1) & 1u);
                tc_fence_after();
                const uint32_t src = tmem + ((uint32_t)(kw * 32) << 16) + rb * S::NT;
#pragma unroll
                for (int c0 = 0; c0 < S::NT; c0 += 48) {
                    uint32_t v[3][16];
#pragma unroll
                    for (int t = 0; t < 3; ++t)
                        if (c0 + 16 * t < S::NT) tmem_ld16(src + c0 + 16 * t, v[t]);
                    tmem_wait_ld();
#pragma unroll
                    for (int t = 0; t < 3; ++t)
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c0 + 16 * t < S::NT) racc[c0 + 16 * t + i] += __uint_as_float(v[t][i]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&rempty[rb]);
            };
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                int r = u / p.n_wt;
                const int qc = r % p.n_qc;
                const int q0 = qc * p.q_chunk, q1 = min(p.Qout, q0 + p.q_chunk);
                for (int s = 0; s < q1 - q0; ++s) {
                    for (int dp = 0; dp < NXP; ++dp,   // G3: the row's 3 dY parts
                         (++didx == (uint32_t)p.nd ? (didx = 0u, dph ^= 1u) : 0u),
                         (++aidx == (uint32_t)p.na ? (aidx = 0u, aph ^= 1u) : 0u)) {
                    mbar_wait(&dfull[didx], dph);
                    mbar_wait(&aempty[aidx], aph ^ 1);
                    tc_fence_after();
                    const uint32_t src = smem_u32(dring + (size_t)didx * kTsDSlot);
                    const uint32_t dst = tmem + ((uint32_t)(32 * kw) << 16) + ACOL + aidx * S::ACOLS;
                    static_assert(kTsKT == 8, "one x16 store covers the 8 K steps of a tile");
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (p.dbg & 1) break;
                        uint32_t v[kTsKT][4];
#pragma unroll
                        for (int ks = 0; ks < kTsKT; ++ks) {
                            const int row = rbase + ks * 16;
                            const uint32_t a = src + h * kTsDHalf + row * kTsDRow +
                                               ((chunk ^ ((row >> 2) & 1)) << 4);
                            ldsm_x4_trans(a, v[ks]);
                        }
                        tmem_st_16x128b_x16(dst + ((uint32_t)(16 * h) << 16), v);
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&dempty[didx]);
                        mbar_arrive(&afull[aidx]);
                    }
                    }   // parts
                    if constexpr (RF) {   // the previous group's MMAs overlap this row's A
                        if (rrow > 0 && (rrow & ((1u << p.rf_shift) - 1u)) == 0)
                            drain(rrow / (1u << p.rf_shift) - 1u);
                        ++rrow;
                    }
                }
            }
            if constexpr (RF) {
                if (rrow > 0) drain(((rrow - 1) >> p.rf_shift));
                float *dst = p.partial + ((size_t)blockIdx.x * 96 + kw * 32 + lane) * S::NT;
#pragma unroll
                for (int c = 0; c < S::NT; c += 4)
                    *reinterpret_cast<float4 *>(dst + c) =
                        make_float4(racc[c], racc[c + 1], racc[c + 2], racc[c + 3]);
            } else {
            // epilogue: D rows (kw, co) of this warp's lane quarter -> per-CTA partial
            mbar_wait(done, 0);
            tc_fence_after();
            float *dst = p.partial + ((size_t)blockIdx.x * 96 + kw * 32 + lane) * S::NT;
#pragma unroll 1
            for (int c = 0; c < S::NT; c += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(kw * 32) << 16) + c, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4 *>(dst + c + i) =
                        make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                    __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// dw[co][ci][kp][kq][kw] = sum_cta partial[cta][kw*32 + co][(kq*KP + kp)*Cin + ci]
// Sum of the per-CTA partials [cta][96][NT] into dW.  A block covers 32
// consecutive partial columns (coalesced 128-B reads) with 8 warps, warp g
// summing CTAs g, g + 8, ... (four independent loads in flight per step),
// then the 8 partial sums are added in a fixed order: deterministic, and
// the loads no longer sit behind one serial 148-term dependency chain per
// thread (was ~41 us per call, latency-bound).
__global__ void __launch_bounds__(kRedCols * kRedGroups)
wgrad_ts_reduce(const float *__restrict__ part, float *__restrict__ dw, int ctas, int KP, int Cin) {
    __shared__ double red[kRedGroups][kRedCols + 1];
    const int KQ = 3, KW = 3;
    const int NT = KQ * KP * Cin;
    const int total = 96 * NT;            // partial layout order: coalesced reads
    const size_t per_cta = (size_t)total;
    const int lo = threadIdx.x % kRedCols, g = threadIdx.x / kRedCols;
    const int o = blockIdx.x * kRedCols + lo;
    double s = 0.0;   // fp64: exact enough for any CTA count
    if (o < total) {
        int c = g;
        for (; c + 3 * kRedGroups < ctas; c += 4 * kRedGroups) {
            const float a0 = part[(size_t)c * per_cta + o];
            const float a1 = part[(size_t)(c + kRedGroups) * per_cta + o];
            const float a2 = part[(size_t)(c + 2 * kRedGroups) * per_cta + o];
            const float a3 = part[(size_t)(c + 3 * kRedGroups) * per_cta + o];
            s += (double)a0;
            s += (double)a1;
            s += (double)a2;
            s += (double)a3;
        }
        for (; c < ctas; c += kRedGroups) s += (double)part[(size_t)c * per_cta + o];
    }
    red[g][lo] = s;
    __syncthreads();
    if (g == 0 && o < total) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < kRedGroups; ++k) t += red[k][lo];
        const int kwco = o / NT, col = o % NT;
        const int kw = kwco / 32, co = kwco % 32;
        const int ci = col % Cin, kqkp = col / Cin;
        const int kp = kqkp % KP, kq = kqkp / KP;
        dw[(((co * Cin + ci) * KP + kp) * KQ + kq) * KW + kw] = (float)t;
    }
}

struct TsPlan {
    Roles R;
    int Cin, nt, xslot, nx, nd, na, smem, grid, q_chunk, n_qc, w_lo, n_wt;
    bool rf;   // row flush (two-level fp32 accumulation, the bf16x3 fp32 wgrad)
    int64_t n_units;
};

bool ts_disabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DP_WGRAD_TS");
        v = (e && e[0] == '0') ? 1 : 0;
    }
    return v == 1;
}

// g3: the grouped bf16x3 wgrad (all 6 part pairings per unit, conv_wgrad_ts_kernel G3)
bool make_tsplan(const dp_conv_geom *g, TsPlan &pl, bool fp32 = false, bool g3 = false) {
    if (ts_disabled()) return false;
    if (!map_roles(g, false, pl.R)) return false;
    const Roles &R = pl.R;
    pl.Cin = (int)g->c_in;
    if (g->c_out != kTsCo || R.KQ != 3 || R.KW != 3) return false;
    const bool ok = (R.KP == 3 && (pl.Cin == 16 || pl.Cin == 32)) ||
                    (R.KP == 1 && (pl.Cin == 16 || pl.Cin == 32 || pl.Cin == 64));
    if (!ok) return false;
    if (g->xs[1] != 1 || g->ys[1] != 1) return false;
    if (g->halo > 0 && g->hs[1] != 1) return false;
    for (int i = 0; i < 4; ++i) {
        if (R.xs[i] % 8 || R.ys[i] % 8) return false;
        if (g->halo > 0 && R.hs[i] % 8) return false;
    }
    const int cbx = chan_block(pl.Cin);
    pl.nt = 3 * R.KP * pl.Cin;
    pl.rf = fp32 && pl.nt <= 96;
    if (g3 && !(pl.rf && R.KP == 1 && pl.Cin == 32)) return false;
    pl.xslot = R.KP * (pl.Cin / cbx) * kTsWK * cbx * 2 * (g3 ? 3 : 1);
    const int acol = ((pl.rf ? 2 : 1) * pl.nt + 31) / 32 * 32;
    pl.na = (512 - acol) / (kTsKT * 8);
    static const int na_cap = getenv("DP_WGRAD_NA") ? atoi(getenv("DP_WGRAD_NA")) : 4;
    if (!g3 && pl.na > na_cap) pl.na = na_cap;   // G3: 3 A entries per row, take them all
    if (pl.na < (g3 ? 3 : 2)) return false;
    const int budget = 220 * 1024 - 512;
    static const int nd = getenv("DP_WGRAD_ND") ? atoi(getenv("DP_WGRAD_ND")) : 4;
    pl.nd = g3 ? 6 : nd;                          // G3: two rows of 3 dY parts
    pl.nx = (budget - pl.nd * kTsDSlot) / pl.xslot;
    // X ring depth (L1 wgrad 0.504 -> 0.494 ms at 12, measured with mirrored slots)
    static const int nx_cap = getenv("DP_WGRAD_NX") ? atoi(getenv("DP_WGRAD_NX")) : 12;
    if (pl.nx > nx_cap) pl.nx = nx_cap;
    if (pl.nx < 4) return false;
    pl.smem = pl.nx * pl.xslot + pl.nd * kTsDSlot + 512;
    // useful w' columns: X real there (padding columns contribute zero)
    const int wr = R.Wout + 3 - 1;
    pl.w_lo = R.base_w < 0 ? -R.base_w : 0;
    int w_hi = R.Win - R.base_w;
    if (w_hi > wr) w_hi = wr;
    pl.n_wt = w_hi > pl.w_lo ? (w_hi - pl.w_lo + kTsWK - 1) / kTsWK : 0;
    const int sms = sm_count();
    const int64_t cols = (int64_t)g->batch * R.Pout * pl.n_wt;
    int best_chunk = R.Qout > 0 ? R.Qout : 1;
    double best = -1;
    for (int nq = 1; nq <= R.Qout && nq <= 64; ++nq) {
        const int chunk = (R.Qout + nq - 1) / nq;
        const int nqc = (R.Qout + chunk - 1) / chunk;
        const int64_t units = cols * nqc;
        const int64_t waves = (units + sms - 1) / sms;
        const double balance = (double)units / (double)(waves * sms);
        const double overhead = (double)(chunk + 2) / chunk;
        const double score = balance / overhead;
        if (score > best + 1e-9) {
            best = score;
            best_chunk = chunk;
        }
    }
    pl.q_chunk = best_chunk;
    pl.n_qc = R.Qout > 0 ? (R.Qout + best_chunk - 1) / best_chunk : 0;
    pl.n_units = cols * pl.n_qc;
    pl.grid = (int)(pl.n_units < sms ? pl.n_units : sms);
    if (pl.grid < 1) pl.grid = 1;
    return true;
}

int64_t ts_workspace(const TsPlan &pl) { return (int64_t)pl.grid * 96 * pl.nt * 4; }

template <int CIN, int KP, bool RF = false, bool G3 = false>
int launch_ts_k(const CUtensorMap &xm, const CUtensorMap &hm, const CUtensorMap &dm,
                const WgradTsParams &p, int grid, int smem, cudaStream_t st) {
    auto kern = conv_wgrad_ts_kernel<CIN, KP, RF, G3>;
    DP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, st>>>(xm, hm, dm, p);
    return launch_status("conv_wgrad_ts_kernel");
}

int run_wgrad_ts(const dp_conv_geom *g, const TsPlan &pl, const void *x, const void *xh,
                 const void *dy, float *dw, void *ws, int64_t ws_bytes, cudaStream_t st,
                 int pairB = 0, bool g3 = false) {
    const uint64_t nb = pairB > 0 ? (uint64_t)3 * pairB : (uint64_t)g->batch;   // tensor batch
    const Roles &R = pl.R;
    DP_REQUIRE(ws_bytes >= ts_workspace(pl), DP_ERR_INVALID, "conv_wgrad_ts: workspace too small");
    const int taps = R.KP * 9;
    if (pl.n_units == 0) {
        DP_CUDA_CHECK(cudaMemsetAsync(dw, 0, (size_t)kTsCo * pl.Cin * taps * 4, st));
        return DP_OK;
    }
    const int cbx = chan_block(pl.Cin);
    const CUtensorMapSwizzle sw = cbx == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : cbx == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
    uint32_t xbox[5] = {(uint32_t)cbx, (uint32_t)kTsWK, 1, 1, 1};
    CUtensorMap xm, hm, dm;
    {
        uint64_t dims[5] = {(uint64_t)pl.Cin, (uint64_t)R.Win, (uint64_t)R.Qin, (uint64_t)R.Pin,
                            nb};
        uint64_t strides[4] = {(uint64_t)R.xs[3] * 2, (uint64_t)R.xs[2] * 2,
                               (uint64_t)R.xs[1] * 2, (uint64_t)R.xs[0] * 2};
        int rc = encode_tensor_map(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(x),
                                   dims, strides, xbox, sw);
        if (rc) return rc;
    }
    hm = xm;
    if (g->halo > 0) {
        uint64_t dims[5] = {(uint64_t)pl.Cin, (uint64_t)R.Win,
                            (uint64_t)(R.split == 1 ? g->halo : R.Qin),
                            (uint64_t)(R.split == 0 ? g->halo : R.Pin), nb};
        uint64_t strides[4] = {(uint64_t)R.hs[3] * 2, (uint64_t)R.hs[2] * 2,
                               (uint64_t)R.hs[1] * 2, (uint64_t)R.hs[0] * 2};
        int rc = encode_tensor_map(&hm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                                   const_cast<void *>(xh), dims, strides, xbox, sw);
        if (rc) return rc;
    }
    {
        uint64_t dims[5] = {(uint64_t)kTsCo, (uint64_t)R.Wout, (uint64_t)R.Qout, (uint64_t)R.Pout,
                            nb};
        uint64_t strides[4] = {(uint64_t)R.ys[3] * 2, (uint64_t)R.ys[2] * 2,
                               (uint64_t)R.ys[1] * 2, (uint64_t)R.ys[0] * 2};
        uint32_t dbox[5] = {16, (uint32_t)(kTsWK + 2), 1, 1, 1};
        int rc = encode_tensor_map(&dm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(dy),
                                   dims, strides, dbox, CU_TENSOR_MAP_SWIZZLE_32B);
        if (rc) return rc;
    }
    WgradTsParams p;
    memset(&p, 0, sizeof(p));
    p.Pin = R.Pin; p.Qin = R.Qin; p.Win = R.Win;
    p.Pout = R.Pout; p.Qout = R.Qout; p.Wout = R.Wout;
    p.base_p = R.base_p; p.base_q = R.base_q; p.base_w = R.base_w;
    p.split = g->halo > 0 ? R.split : -1;
    p.halo = (int)g->halo;
    p.w_lo = pl.w_lo; p.n_wt = pl.n_wt; p.n_qc = pl.n_qc; p.q_chunk = pl.q_chunk;
    p.n_units = (int)pl.n_units;
    p.nx = pl.nx; p.nd = pl.nd; p.na = pl.na;
    p.partial = (float *)ws;
    p.pairB = pairB;
    // RF flush group: rows the tensor core accumulates before the round-to-
    // nearest register add (DP_WGRAD_RF_ROWS, a power of two; measured on the
    // full cfg1 grid vs fp64: 1 row 3.9e-7, 4 rows 5.9e-7, 8 rows 1.1e-6 of
    // max|dW| — the reference's bound is 1e-5 — and 0.178 -> 0.162 ms)
    // G3 (all 6 pairings in one tile, small products first): one row per group —
    // 2.0e-7 of max|dW| on cfg1 at 0.1375 ms, vs 2.9e-6 at 0.134 ms with 4 rows
    // (and 5.9e-7 / 0.152 ms for the pairings as batch entries with 4 rows)
    static const int rf_env = getenv("DP_WGRAD_RF_ROWS") ? atoi(getenv("DP_WGRAD_RF_ROWS")) : 0;
    const int rf_rows = rf_env > 0 ? rf_env : (g3 ? 1 : 4);
    p.rf_shift = 0;
    while ((2 << p.rf_shift) <= rf_rows && p.rf_shift < 5) ++p.rf_shift;
    static const int dbg = getenv("DP_CONV_DBG") ? atoi(getenv("DP_CONV_DBG")) : 0;
    p.dbg = dbg;
    int rc;
    if (g3)
        rc = launch_ts_k<32, 1, true, true>(xm, hm, dm, p, pl.grid, pl.smem, st);
    else if (R.KP == 3)
        rc = pl.Cin == 16 ? launch_ts_k<16, 3>(xm, hm, dm, p, pl.grid, pl.smem, st)
                          : launch_ts_k<32, 3>(xm, hm, dm, p, pl.grid, pl.smem, st);
    else if (pl.rf)
        rc = pl.Cin == 16 ? launch_ts_k<16, 1, true>(xm, hm, dm, p, pl.grid, pl.smem, st)
                          : launch_ts_k<32, 1, true>(xm, hm, dm, p, pl.grid, pl.smem, st);
    else
        rc = pl.Cin == 16   ? launch_ts_k<16, 1>(xm, hm, dm, p, pl.grid, pl.smem, st)
             : pl.Cin == 32 ? launch_ts_k<32, 1>(xm, hm, dm, p, pl.grid, pl.smem, st)
                            : launch_ts_k<64, 1>(xm, hm, dm, p, pl.grid, pl.smem, st);
    if (rc) return rc;
    const int total = 96 * 3 * R.KP * pl.Cin;
    wgrad_ts_reduce<<<(unsigned)((total + kRedCols - 1) / kRedCols), kRedCols * kRedGroups, 0, st>>>(
        (const float *)ws, dw, pl.grid, R.KP, pl.Cin);
    return launch_status("wgrad_ts_reduce");
}

}  // namespace

int encode_tensor_map(CUtensorMap *map, CUtensorMapDataType dtype, int rank, void *base,
                      const uint64_t *dims, const uint64_t *strides_bytes, const uint32_t *box,
                      CUtensorMapSwizzle swizzle) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        DP_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
        DP_REQUIRE(ptr && q == cudaDriverEntryPointSuccess, DP_ERR_CUDA,
                   "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    // L2 sector promotion of the TMA reads (DP_TMA_PROMO = 0 / 64 / 128 / 256)
    static int promo = -1;
    if (promo < 0) {
        const char *e = getenv("DP_TMA_PROMO");
        promo = e ? atoi(e) : 128;
    }
    const CUtensorMapL2promotion pr = promo >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                      : promo >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                      : promo >= 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                                    : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    CUresult r = fn(map, dtype, rank, base, dims, strides_bytes, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DP_REQUIRE(r == CUDA_SUCCESS, DP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return DP_OK;
}

int conv_tc_eligible(const dp_conv_geom *g, int dtype, int which) {
    if (dtype != DP_BF16 || !g) return 0;
    if (which == DP_CONV_WGRAD) {
        TsPlan tp;
        WPlan wp;
        return (make_tsplan(g, tp) || make_wplan(g, wp)) ? 1 : 0;
    }
    Plan pl;
    return make_plan(g, which == DP_CONV_DGRAD, pl) ? 1 : 0;
}

int64_t conv_tc_workspace(const dp_conv_geom *g, int which) {
    if (which == DP_CONV_WGRAD) {
        TsPlan tp;
        if (make_tsplan(g, tp)) return ts_workspace(tp);
        WPlan wp;
        if (!make_wplan(g, wp)) return -1;
        return (int64_t)wp.grid * wp.n_mt * 128 * wp.R.KW * wp.N * 4;
    }
    Plan pl;
    if (!make_plan(g, which == DP_CONV_DGRAD, pl)) return -1;
    return 2 * (int64_t)pl.wimg_bytes;   // room for the CTA-pair image ([2][...])
}

// bf16x3 fp32 wgrad (conv_x3.cu): x / dy hold 3 parts each as batch blocks
// [3B]; the 6 pairings run as batch entries of g (g->batch = 6B)
// The grouped form (G3: units over the B real batch entries, each running all
// 6 pairings) when the shape has it; DP_WGRAD_G3=0 keeps the pairings as
// batch entries.
bool x3_g3_plan(const dp_conv_geom *g, int B, dp_conv_geom &g1, TsPlan &tp) {
    static const bool off = getenv("DP_WGRAD_G3") && getenv("DP_WGRAD_G3")[0] == '0';
    if (off || B <= 0 || g->batch != 6 * (int64_t)B) return false;
    g1 = *g;
    g1.batch = B;
    return make_tsplan(&g1, tp, true, true);
}
int conv_wgrad_x3_launch(const dp_conv_geom *g, const void *x, const void *xh, const void *dy,
                         void *dw, void *ws, int64_t ws_bytes, cudaStream_t st, int B) {
    TsPlan tp;
    dp_conv_geom g1;
    if (x3_g3_plan(g, B, g1, tp))
        return run_wgrad_ts(&g1, tp, x, xh, dy, (float *)dw, ws, ws_bytes, st, B, true);
    DP_REQUIRE(make_tsplan(g, tp, true), DP_ERR_UNSUPPORTED, "conv_wgrad_x3: outside the envelope");
    return run_wgrad_ts(g, tp, x, xh, dy, (float *)dw, ws, ws_bytes, st, B);
}
int64_t conv_wgrad_x3_workspace(const dp_conv_geom *g) {
    TsPlan tp;
    if (!make_tsplan(g, tp, true)) return -1;
    int64_t ws = ts_workspace(tp);
    dp_conv_geom g1;
    TsPlan t3;
    if (g->batch % 6 == 0 && x3_g3_plan(g, (int)(g->batch / 6), g1, t3) && ts_workspace(t3) > ws)
        ws = ts_workspace(t3);
    return ws;
}

// bf16 tcgen05 conv with fp32 outputs (the bf16x3 fp32 path, conv_x3.cu)
int64_t conv_tc_f32out_workspace(const dp_conv_geom *g, bool dgrad) {
    Plan pl;
    return make_plan(g, dgrad, pl, true, true) ? 2 * (int64_t)pl.wimg_bytes : -1;
}
// g describes the 6-block MMA view (c_in or c_out = 6 C); the activation
// operand holds the 3 parts once as batch blocks [3][B][..][C] (strides in g
// are those of one [B][..][C] block)
int conv_tc_f32out_launch(const dp_conv_geom *g, bool dgrad, const void *in, const void *in_halo,
                          const void *w, void *out, void *out2, void *ws, int64_t ws_bytes,
                          cudaStream_t st) {
    return run_conv_tc(g, dgrad, in, in_halo, w, out, out2, ws, ws_bytes, st, true, true);
}

int conv_fwd_tc_launch(const dp_conv_geom *g, const void *x, const void *xh, const void *w, void *y,
                       void *ws, int64_t ws_bytes, cudaStream_t st) {
    return run_conv_tc(g, false, x, xh, w, y, nullptr, ws, ws_bytes, st);
}

int conv_dgrad_tc_launch(const dp_conv_geom *g, const void *dy, const void *w, void *dx, void *dxh,
                         void *ws, int64_t ws_bytes, cudaStream_t st) {
    return run_conv_tc(g, true, dy, nullptr, w, dx, dxh, ws, ws_bytes, st);
}

int conv_wgrad_tc_launch(const dp_conv_geom *g, const void *x, const void *xh, const void *dy,
                         void *dw, void *ws, int64_t ws_bytes, cudaStream_t st) {
    TsPlan tp;
    if (make_tsplan(g, tp)) return run_wgrad_ts(g, tp, x, xh, dy, (float *)dw, ws, ws_bytes, st);
    return run_wgrad_tc(g, x, xh, dy, (float *)dw, ws, ws_bytes, st);
}

}  // namespace dp
