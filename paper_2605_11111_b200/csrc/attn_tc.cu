// tcgen05 + TMA ring-attention block kernels (bf16 in, fp32 state), head
// dim 64.  One launch folds ONE K/V block of the ring into the running
// online-softmax state (m, l, acc) of the local queries — the reference's
// per-step `scores = q @ kb.T * scale; state.update(scores, vb)`
// (domainpar/ops.py:272-275, RingSoftmaxState.update :199-211) — so the ring
// loop on the host (K||V rotating over NVLink) is unchanged; the state
// stays fp32 in HBM between ring steps.
//
// Forward (attn_fwd_tc_kernel): CTA = TWO 128-row query tiles of one head,
// looping over the block's keys 128 at a time; 384 threads:
//   warpgroup 0  warp 0 TMA producer (Q once, K/V tiles into a 4-stage
//                ring), warp 1 MMA issuer: S_t(j) = Q_t K_j^T (SS, M=128,
//                N=128, K=64) and O_t += P_t(j) V_j (TS: P from TMEM, V as
//                the MN-major smem B operand, M=128, N=64, K=128) for both
//                tiles t, ping-ponging between the two softmax warpgroups
//   warpgroups 1-2  softmax of tile t (thread = query row = TMEM lane):
//                tcgen05.ld its S row, online max with lazy rescaling (O and
//                l rescaled only when the row max grows by > 2^8: exact, any
//                reference max gives the same acc/l), P = exp2(.) written as
//                packed bf16 pairs into its own TMEM columns (no smem round
//                trip); POLY exp2 pairs in eight on the FMA pipe (cubic);
//                they load acc into TMEM at the start and write the state
//                (m, l, acc; LSE for the backward) back at the end.
// TMEM per tile: S [128 t, +128), P [256 + 64 t, +64), O [384 + 64 t, +64);
// P does not alias S, so S_t(j+1) is issued as soon as the softmax has read
// S_t(j).  setmaxnreg splits registers 80 (warpgroup 0) / 208 (softmax).
//
// Backward (attn_bwd_tc_kernel): CTA = one 128-key tile (K, V resident, dK
// and dV accumulated in TMEM) looping over 128-row query blocks (Q, dO in a
// 3-stage TMA ring); 768 threads in six warpgroups: S^T = K Q^T and
// dP^T = V dO^T into TMEM, 16 softmax warps write P^T as bf16 pairs into TMEM
// (the TS A operand of dV += P^T dO) and dS^T = scale P^T o (dP^T - D) as a
// swizzled smem tile (double-buffered) for dK += dS^T Q and dQ = dS K; dQ is
// drained by 4 epilogue warps through swizzled fp32 smem and a TMA bulk
// reduce-add into dq, and the same warps stage -LSE*log2e / scale*D rows into
// a smem ring two blocks ahead.
// Operand layouts: Q, K, V, dO tiles land from TMA as [128 rows][64 d] with
// the 128-B swizzle.
#include "tc_common.cuh"
#include <cstdio>

namespace dp {
namespace {

constexpr int kBM = 128;      // query rows per tile
constexpr int kBN = 128;      // keys per block
constexpr int kD = 64;        // head dim
constexpr int kStages = 3;    // K/V ring depth
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.0f;  // log2 units: rescale when the max grows by > 2^8

constexpr int kTileBytes = kBM * kD * 2;           // 16 KB (Q, K or V tile)
constexpr int kPBytes = kBM * kBN * 2;             // 32 KB (P tile)

// Forward: two 128-row query tiles per CTA (two softmax warpgroups that
// ping-pong against the single MMA warp).
constexpr int kFwdTiles = 2;
constexpr int kFwdThreads = 128 + 128 * kFwdTiles;  // WG0: TMA + MMA warps; WG1..: softmax
constexpr int kFwdStages = 4;                              // K/V ring depth
constexpr int kSmemQ = 0;
constexpr int kSmemKV = kSmemQ + kFwdTiles * kTileBytes;  // stages of [K | V]
constexpr int kSmemBar = kSmemKV + kFwdStages * 2 * kTileBytes;
constexpr int kSmemFwd = kSmemBar + 256;

// TMEM columns per tile t: S_t [128 t, +128), P_t (bf16 pairs) [256 + 64 t,
// +64), O_t [384 + 64 t, +64).  P has its own columns so S_t(j+1) can be
// computed while the softmax still works on block j (Q stays in smem: the S
// MMA is SS, 64 cycles per K step either way).
constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;

struct FwdParams {
    int sq, sk, H;
    int n_qt;                 // CTAs per head (kFwdTiles query tiles each)
    float c;                  // scale * log2(e)
    float *m, *l, *acc;       // fp32 state: [sq,H], [sq,H], [sq,H,64]
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// packed fp32x2 FMA / add (sm_100 FFMA2 / FADD2): two scores per instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)),
          "l"(*reinterpret_cast<unsigned long long *>(&c)));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("add.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)));
    return d;
}

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("mul.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)));
    return d;
}

// exp2 of two arguments on the FMA pipe (FA4-style MUFU offload): round to
// nearest via the 1.5*2^23 magic constant, a cubic for 2^f on [-1/2, 1/2]
// (max rel err 1.1e-4, far below the bf16 rounding of P), exponent bits
// added with one integer multiply-add.  Arguments are <= 2^kRescale-bounded
// from above; very negative ones flush to 0 through the clamp.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    const float2 lo = make_float2(-127.f, -127.f);
    x.x = fmaxf(x.x, lo.x);
    x.y = fmaxf(x.y, lo.y);
    const float2 M = make_float2(12582912.f, 12582912.f);
    const float2 t = fadd2(x, M);
    const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = fadd2(x, make_float2(-j.x, -j.y));
    float2 pp = ffma2(make_float2(0.05459282f, 0.05459282f), f,
                      make_float2(0.24221784f, 0.24221784f));
    pp = ffma2(pp, f, make_float2(0.6933686f, 0.6933686f));
    pp = ffma2(pp, f, make_float2(1.f, 1.f));
    float2 r;
    r.x = __int_as_float(__float_as_int(pp.x) + (__float_as_int(t.x) << 23));
    r.y = __int_as_float(__float_as_int(pp.y) + (__float_as_int(t.y) << 23));
    return r;
}

template <int POLY>  // exp2 pairs of every 8 computed on the FMA pipe instead of MUFU
__global__ void __launch_bounds__(kFwdThreads, 1)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                   const __grid_constant__ CUtensorMap vmap, const FwdParams p) {
    using namespace tc;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);   // warp-uniform for ptxas
    const int lane = threadIdx.x & 31;
    const int qt = blockIdx.x % p.n_qt, h = blockIdx.x / p.n_qt;
    const int q0 = qt * kBM * kFwdTiles;
    const int nblk = (p.sk + kBN - 1) / kBN;

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kSmemBar);
    uint64_t *q_full = bars;
    uint64_t *kv_full = bars + 1, *kv_empty = kv_full + kFwdStages;
    uint64_t *s_full = kv_empty + kFwdStages;   // [tiles]  S_t(j) ready
    uint64_t *s_free = s_full + kFwdTiles;      // [tiles]  softmax loaded S_t(j) (count 128)
    uint64_t *p_full = s_free + kFwdTiles;      // [tiles]  P_t(j) written (count 128)
    uint64_t *pv_done = p_full + kFwdTiles;     // [tiles]  PV_t(j) finished (O, P_t quiescent)
    uint64_t *done = pv_done + kFwdTiles;       // every MMA finished
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    if (warp == 0) {
        if (lane == 0) {
            mbar_init(q_full, 1);
            for (int i = 0; i < kFwdStages; ++i) {
                mbar_init(&kv_full[i], 1);
                mbar_init(&kv_empty[i], 1);
            }
            for (int i = 0; i < kFwdTiles; ++i) {
                mbar_init(&s_full[i], 1);
                mbar_init(&s_free[i], 128);
                mbar_init(&p_full[i], 128);
                mbar_init(&pv_done[i], 1);
            }
            mbar_init(done, 1);
            mbar_fence_init();
            tma_prefetch(&qmap);
            tma_prefetch(&kmap);
            tma_prefetch(&vmap);
        }
        __syncwarp();
        tmem_alloc_ool(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // Registers: the softmax warpgroups hold a 128-score row each; the
    // producer warpgroup needs few.  setmaxnreg moves the budget (per SMSP:
    // 80 + 208 + 208 regs x 32 lanes fits the 16K-register sub-partition).
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;");
    if (warp == 0) {
        // ===================== TMA producer =====================
        mbar_expect_tx_e(q_full, kFwdTiles * kTileBytes);
        for (int t = 0; t < kFwdTiles; ++t)
            tma_load_3d_e(smem + kSmemQ + t * kTileBytes, &qmap, q_full, 0, h, q0 + t * kBM);
        for (int j = 0; j < nblk; ++j) {
            const int st = j % kFwdStages;
            mbar_wait(&kv_empty[st], ((j / kFwdStages) & 1) ^ 1);
            mbar_expect_tx_e(&kv_full[st], 2 * kTileBytes);
            uint8_t *dst = smem + kSmemKV + st * 2 * kTileBytes;
            tma_load_3d_e(dst, &kmap, &kv_full[st], 0, h, j * kBN);
            tma_load_3d_e(dst + kTileBytes, &vmap, &kv_full[st], 0, h, j * kBN);
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        // S_t = Q_t K^T (SS, Q from smem), O_t += P_t V with P_t in TMEM (TS).
        // S_t(j+1) is issued as soon as softmax t has LOADED S_t(j) (s_free),
        // so it runs under that softmax; PV_t(j) follows P_t(j) (p_full).
        const uint32_t id_s = idesc_bf16(kBM, kBN);            // K-major A, K-major B
        const uint32_t id_o = idesc_bf16(kBM, kD, 0, 1);       // P K-major, V MN-major
        mbar_wait(q_full, 0);
        auto issue_s = [&](int t, int j) {
            const int st = j % kFwdStages;
            const uint64_t kd = sdesc_sw(smem_u32(smem + kSmemKV + st * 2 * kTileBytes), 1024, 2);
            const uint64_t qd = sdesc_sw(smem_u32(smem + kSmemQ + t * kTileBytes), 1024, 2);
            const uint32_t sc = tmem + kColS + t * kBN;
#pragma unroll
            for (int k = 0; k < kD / 16; ++k)
                mma_bf16_e(sc, qd + ((k * 32) >> 4), kd + ((k * 32) >> 4), id_s, k ? 1u : 0u);
            mma_commit_e(&s_full[t]);
        };
        auto issue_pv = [&](int t, int j) {
            const int st = j % kFwdStages;
            const uint64_t vd =
                sdesc_mn(smem_u32(smem + kSmemKV + st * 2 * kTileBytes + kTileBytes), 8192, 1024, 2);
#pragma unroll
            for (int k = 0; k < kBN / 16; ++k) {
                const uint32_t vb = (k * 16 * 128) >> 4;  // 16 key rows of V
                mma_ts_e(tmem + kColO + t * kD, tmem + kColP + t * (kBN / 2) + k * 8, vd + vb, id_o, 1u);
            }
            mma_commit_e(&pv_done[t]);
        };
        if (nblk >= 1) {
            mbar_wait(&kv_full[0], 0);
            tc_fence_after();
            for (int t = 0; t < kFwdTiles; ++t) issue_s(t, 0);
        }
        for (int j = 0; j < nblk; ++j) {
            const bool more = j + 1 < nblk;
            if (more) mbar_wait(&kv_full[(j + 1) % kFwdStages], ((j + 1) / kFwdStages) & 1);
            for (int t = 0; t < kFwdTiles; ++t) {
                if (more) {
                    mbar_wait(&s_free[t], j & 1);      // softmax t holds S_t(j) in registers
                    tc_fence_after();
                    issue_s(t, j + 1);
                }
                mbar_wait(&p_full[t], j & 1);
                tc_fence_after();
                issue_pv(t, j);
            }
            mma_commit_e(&kv_empty[j % kFwdStages]);
        }
        mma_commit_e(done);
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
        // ===================== softmax / state (two warpgroups) =====================
        const int t = (warp - 4) >> 2;               // query tile of this warpgroup
        const int quarter = warp & 3;
        const int rl = quarter * 32 + lane;          // row within the tile = TMEM lane
        const int row = q0 + t * kBM + rl;
        const bool valid = row < p.sq;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t colS = lane_base + kColS + t * kBN, colO = lane_base + kColO + t * kD;
        const uint32_t colP = lane_base + kColP + t * (kBN / 2);
        const size_t sidx = (size_t)row * p.H + h;
        float m_run = -INFINITY, l_run = 0.f;
        {
            uint32_t o[16];
            for (int c = 0; c < kD; c += 16) {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    o[i] = valid ? __float_as_uint(p.acc[sidx * kD + c + i]) : 0u;
                tmem_st16(colO + c, o);
            }
            tmem_wait_st();
            if (valid) {
                m_run = p.m[sidx] * kLog2e;
                l_run = p.l[sidx];
            }
        }
        const float2 c2 = make_float2(p.c, p.c);
        for (int j = 0; j < nblk; ++j) {
            mbar_wait(&s_full[t], j & 1);
            tc_fence_after();
            float s[kBN];
#pragma unroll
            for (int c = 0; c < kBN; c += 16) {
                uint32_t u[16];
                tmem_ld16(colS + c, u);
#pragma unroll
                for (int i = 0; i < 16; ++i) s[c + i] = __uint_as_float(u[i]);
            }
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&s_free[t]);            // S_t may be overwritten by S_t(j+1)
            const int kvalid = p.sk - j * kBN;  // keys of this block that exist
            if (kvalid < kBN) {
#pragma unroll
                for (int i = 0; i < kBN; ++i)
                    if (i >= kvalid) s[i] = -INFINITY;
            }
            // row max: 8 independent chains (ILP), then a small tree
            float mq[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) mq[a] = fmaxf(s[a], s[a + 8]);
#pragma unroll
            for (int i = 16; i < kBN; i += 16)
#pragma unroll
                for (int a = 0; a < 8; ++a) mq[a] = fmaxf(mq[a], fmaxf(s[i + a], s[i + 8 + a]));
            const float mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                                   fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7])));
            const float tnew = mx * p.c;
            // lazy rescale: only when this row's max grows by more than 2^kRescale
            // (O must be quiescent: PV_t(j-1) finished)
            const bool grow = tnew > m_run + kRescale;
            if (__any_sync(0xffffffffu, grow)) {
                if (j >= 1) mbar_wait(&pv_done[t], (j - 1) & 1);
                tc_fence_after();
                const float f = grow ? ex2(m_run - tnew) : 1.f;
                for (int c = 0; c < kD; c += 16) {
                    uint32_t o[16];
                    tmem_ld16(colO + c, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                    tmem_st16(colO + c, o);
                }
                tmem_wait_st();
                if (grow) {
                    l_run *= f;
                    m_run = tnew;
                }
            }
            // P = exp2(s c - m) as bf16 pairs into P_t's TMEM columns (written once
            // PV_t(j-1) has read the previous P_t; it had this whole block's
            // exp math to do so)
            const float2 nm = make_float2(-m_run, -m_run);
            uint32_t pk[kBN / 2];
            float2 sumv[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                              make_float2(0.f, 0.f)};   // 4 independent sum chains
#pragma unroll
            for (int c = 0; c < kBN / 32; ++c) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float2 x = ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), c2, nm);
                    if ((i & 7) < POLY) {
                        x = ex2_poly2(x);
                    } else {
                        x.x = ex2(x.x);
                        x.y = ex2(x.y);
                    }
                    sumv[i & 3] = fadd2(sumv[i & 3], x);
                    pk[c * 16 + i] = pack_bf16(x.x, x.y);
                }
            }
            if (j >= 1) mbar_wait(&pv_done[t], (j - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < kBN / 32; ++c)
                tmem_st16(colP + c * 16, *reinterpret_cast<uint32_t(*)[16]>(pk + c * 16));
            tmem_wait_st();
            const float2 sum2 = fadd2(fadd2(sumv[0], sumv[1]), fadd2(sumv[2], sumv[3]));
            l_run += sum2.x + sum2.y;
            tc_fence_before();
            mbar_arrive(&p_full[t]);
        }
        // final state back to HBM once every MMA has landed
        mbar_wait(done, 0);
        tc_fence_after();
        for (int c = 0; c < kD; c += 16) {
            uint32_t o[16];
            tmem_ld16(colO + c, o);
            tmem_wait_ld();
            if (valid) {
                float4 *dst = reinterpret_cast<float4 *>(p.acc + sidx * kD + c);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    dst[i] = make_float4(__uint_as_float(o[4 * i]), __uint_as_float(o[4 * i + 1]),
                                         __uint_as_float(o[4 * i + 2]), __uint_as_float(o[4 * i + 3]));
            }
        }
        if (valid) {
            p.m[sidx] = m_run / kLog2e;
            p.l[sidx] = l_run;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------
// Backward block: with P = exp(s - lse), D = rowsum(dO * O) (from
// dp_attn_bwd_preprocess):  dV += P^T dO,  dS = P (dO V^T - D),
// dQ += scale dS K,  dK += scale dS^T Q  — the same math as the CUDA-core
// kernels, for one K/V block of the ring.
//
// CTA = one 128-key tile of one head (K, V resident in smem; dK, dV
// accumulate in TMEM over the whole query range), looping over 128-row
// query blocks (Q, dO in a 3-stage TMA ring).  768 threads, six warpgroups
// (setmaxnreg: 64 / 4 x 88 / 64 registers):
//   warp 0     TMA producer
//   warp 1     MMA issuer: S^T = K Q^T and dP^T = V dO^T into TMEM; once the
//              softmax warps have written P^T / dS^T (bf16, swizzled smem):
//              dV += P^T dO, dK += dS^T Q (A = the key-major tiles), and
//              dQ = dS K into a double-buffered TMEM tile (A = the SAME dS^T
//              bytes read as an MN-major operand)
//   warps 2-3  idle
//   warps 4-19 four warps per TMEM lane quarter, each a 32-column quarter of
//              the 128 query columns; thread = (key row, column quarter):
//              P^T = exp2(S^T c - LSE2), dS^T = scale P^T (dP^T - D) -> smem
//              (packed fp32x2 math); at the end dV / dK += TMEM (32-column
//              halves).  Four softmax warps per SM sub-partition (was two)
//              hide the MUFU / TMEM-load latency: 16k block 3.09 -> 2.90 ms
//              together with the 3-stage Q / dO ring
//   warps 20-23 thread = query row: dQ tile TMEM -> swizzled fp32 smem ->
//              TMA bulk reduce-add (cp.reduce.async.bulk.tensor .add) into dq
//              (per-thread float4 atomics cost 34 of 84 ms at 64k); they also
//              stage each query block's -LSE*log2(e) / scale*D rows into a
//              smem ring two blocks ahead (mbarrier hand-off, so the softmax
//              warps never wait on global loads or a CTA-wide barrier)
// The next block's S^T / dP^T MMAs are issued before this block's gradient
// MMAs, so the softmax warps overlap the tensor pipe; a Q / dO stage is
// released once dK has read it (dQ only needs dS and K).
// Debug: DP_ATTN_TRACE=1 prints CTA 0's per-block event clocks (the timeline
// behind these choices), DP_ATTN_DBG=<bits> the ablations listed in BwdParams.
constexpr int kBwdThreads = 768;   // TMA, MMA, 2 idle, 16 softmax warps, 4 dQ warps
constexpr int kB_K = 0, kB_V = kTileBytes;
constexpr int kQDStages = 3;                           // [Q | dO] ring (a stage frees when
                                                       // the block's dK MMAs complete)
constexpr int kB_QD = 2 * kTileBytes;
constexpr int kB_PS = kB_QD + kQDStages * 2 * kTileBytes;  // dS^T x 2 (double buffer)
constexpr int kB_DQ = kB_PS + 2 * kPBytes;             // dQ staging tile (fp32, 2 x 16 KB halves)
constexpr int kDQStage = kBM * kD * 4;                 // 32 KB
constexpr int kLDBufs = 2;                             // -lse2 / scale*D ring (dQ warps -> softmax)
constexpr int kB_LD = kB_DQ + kDQStage;                // -lse2[2][128], delta[2][128]
constexpr int kB_BAR = kB_LD + 2 * kLDBufs * 128 * 4;
constexpr int kSmemBwd = kB_BAR + 256;
static_assert(kSmemBwd <= 232448, "attention bwd smem");
// TMEM columns: S^T [0,128), dP^T [128,256), dV [256,320), dK [320,384), dQ [384,448),
// P^T (bf16 pairs, the TS A operand of dV += P^T dO) [448,512)
constexpr uint32_t kColST = 0, kColDP = 128, kColDV = 256, kColDK = 320, kColDQ = 384,
                   kColPT = 448;

struct BwdParams {
    int sq, sk, H;
    int n_kt;
    float c;                  // scale * log2(e)
    float scale;
    const float *lse, *delta;  // [sq, H]
    float *dq;                 // [sq, H, 64] (atomic +=)
    float *dk, *dv;            // [sk, H, 64] (+=)
    int dbg;                   // DP_ATTN_DBG ablations: 1 no dQ reduce, 2 no softmax math,
                               // 4 no gradient MMAs, 8 no S/dP MMAs
    unsigned long long *trace; // DP_ATTN_TRACE: per-block event clocks of CTA 0 (debug)
};

#define BWD_TRACE(blk, ev)                                                              \
    do {                                                                                \
        if (p.trace && blockIdx.x == 0 && lane == 0 && (blk) >= 0 && (blk) < 64)         \
            p.trace[(blk) * 16 + (ev)] = clock64();                                     \
    } while (0)

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(kBwdThreads, 1)
attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                   const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap dmap,
                   const __grid_constant__ CUtensorMap dqmap, const BwdParams p) {
    using namespace tc;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);   // warp-uniform for ptxas
    const int lane = threadIdx.x & 31;
    const int kt = blockIdx.x % p.n_kt, h = blockIdx.x / p.n_kt;
    const int k0 = kt * kBN;
    const int nq = (p.sq + kBM - 1) / kBM;

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kB_BAR);
    uint64_t *kv_full = bars;
    uint64_t *qd_full = bars + 1, *qd_empty = qd_full + kQDStages;
    uint64_t *s_full = qd_empty + kQDStages, *s_free = s_full + 1;
    uint64_t *p_full = s_free + 1;                          // P^T + dS^T(b) written
    uint64_t *pv_empty = p_full + 2;                        // dV done with P^T (TMEM)
    uint64_t *ds_empty = pv_empty + 1;                      // dK + dQ done with dS^T(b)
    uint64_t *dq_full = ds_empty + 2, *dq_empty = dq_full + 1;
    uint64_t *ld_full = dq_empty + 1, *ld_empty = ld_full + kLDBufs;   // [kLDBufs] each
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(ld_empty + kLDBufs);
    float *lse2_s = reinterpret_cast<float *>(smem + kB_LD);   // [kLDBufs][128]
    float *delta_s = lse2_s + kLDBufs * 128;                   // [kLDBufs][128]

    if (warp == 0) {
        if (lane == 0) {
            mbar_init(kv_full, 1);
            for (int i = 0; i < kQDStages; ++i) {
                mbar_init(&qd_full[i], 1);
                mbar_init(&qd_empty[i], 1);
            }
            for (int i = 0; i < 2; ++i) {
                mbar_init(&p_full[i], 512);
                mbar_init(&ds_empty[i], 1);
            }
            mbar_init(dq_full, 1);
            mbar_init(dq_empty, 128);
            for (int i = 0; i < kLDBufs; ++i) {
                mbar_init(&ld_full[i], 128);   // the dQ warps' threads (one query row each)
                mbar_init(&ld_empty[i], 16);   // one arrival per softmax warp
            }
            mbar_init(s_full, 1);
            mbar_init(s_free, 512);
            mbar_init(pv_empty, 1);
            mbar_fence_init();
            tma_prefetch(&qmap);
            tma_prefetch(&kmap);
            tma_prefetch(&vmap);
            tma_prefetch(&dmap);
            tma_prefetch(&dqmap);
        }
        __syncwarp();
        tmem_alloc_ool(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // registers: 64 for the TMA / MMA warpgroup, 88 for the four softmax
    // warpgroups, 64 for the dQ one (launch: 80 x 768 threads)
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    if (warp == 0) {
        // ===================== TMA producer =====================
        mbar_expect_tx_e(kv_full, 2 * kTileBytes);
        tma_load_3d_e(smem + kB_K, &kmap, kv_full, 0, h, k0);
        tma_load_3d_e(smem + kB_V, &vmap, kv_full, 0, h, k0);
        for (int i = 0; i < nq; ++i) {
            const int st = i % kQDStages;
            mbar_wait(&qd_empty[st], ((i / kQDStages) & 1) ^ 1);
            BWD_TRACE(i, 14);
            if (p.dbg & 16) {
                if (lane == 0) mbar_arrive(&qd_full[st]);
                __syncwarp();
                continue;
            }
            mbar_expect_tx_e(&qd_full[st], 2 * kTileBytes);
            uint8_t *dst = smem + kB_QD + st * 2 * kTileBytes;
            tma_load_3d_e(dst, &qmap, &qd_full[st], 0, h, i * kBM);
            tma_load_3d_e(dst + kTileBytes, &dmap, &qd_full[st], 0, h, i * kBM);
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        const uint32_t id_s = idesc_bf16(kBN, kBM);           // M = keys, N = queries
        const uint32_t id_g = idesc_bf16(kBN, kD, 0, 1);      // dV / dK: A K-major, B MN-major
                                                              // (dV: A = P^T from TMEM, TS)
        const uint32_t id_q = idesc_bf16(kBM, kD, 1, 1);      // dQ: A (dS) MN-major, B MN-major
        const uint64_t kd = sdesc_sw(smem_u32(smem + kB_K), 1024, 2);
        const uint64_t vd = sdesc_sw(smem_u32(smem + kB_V), 1024, 2);
        const uint64_t kmn = sdesc_mn(smem_u32(smem + kB_K), 8192, 1024, 2);
        mbar_wait(kv_full, 0);
        auto issue_grads = [&](int j) {
            const int b = j & 1;
            mbar_wait(&p_full[b], (j >> 1) & 1);
            BWD_TRACE(j, 1);
            tc_fence_after();
            const int qs = j % kQDStages;
            uint8_t *qdst = smem + kB_QD + qs * 2 * kTileBytes;
            uint8_t *ps = smem + kB_PS + b * kPBytes;            // dS^T(b)
            const uint64_t dst_k = sdesc_sw(smem_u32(ps), 1024, 2);
            const uint64_t ds_mn = sdesc_mn(smem_u32(ps), kBM * 128, 1024, 2);
            const uint64_t q_mn = sdesc_mn(smem_u32(qdst), 8192, 1024, 2);
            const uint64_t do_mn = sdesc_mn(smem_u32(qdst + kTileBytes), 8192, 1024, 2);
#pragma unroll
            for (int k = 0; k < kBM / 16; ++k) {   // dV += P^T dO (P^T in TMEM)
                if (p.dbg & 4) break;
                const uint32_t bb = (k * 16 * 128) >> 4;
                mma_ts_e(tmem + kColDV, tmem + kColPT + k * 8, do_mn + bb, id_g,
                         (j > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit_e(pv_empty);                 // the softmax may overwrite P^T
            BWD_TRACE(j, 3);
#pragma unroll
            for (int k = 0; k < kBM / 16; ++k) {   // dK += dS^T Q
                if (p.dbg & 4) break;
                const uint32_t a = ((k >> 2) * (kBN * 128) + (k & 3) * 32) >> 4;
                const uint32_t bb = (k * 16 * 128) >> 4;
                mma_bf16_e(tmem + kColDK, dst_k + a, q_mn + bb, id_g, (j > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit_e(&qd_empty[qs]);            // Q / dO(j) no longer read (dQ uses dS, K)
            BWD_TRACE(j, 8);
            if (j >= 1) mbar_wait(dq_empty, (j - 1) & 1);   // dQ(j-1) drained from TMEM
            BWD_TRACE(j, 2);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < kBN / 16; ++k) {   // dQ = dS K
                if (p.dbg & 4) break;
                const uint32_t a = (k * 16 * 128) >> 4;     // 16 key rows of dS^T
                mma_bf16_e(tmem + kColDQ, ds_mn + a, kmn + a, id_q, k ? 1u : 0u);
            }
            mma_commit_e(&ds_empty[b]);
            mma_commit_e(dq_full);
            BWD_TRACE(j, 11);
        };
        for (int i = 0; i < nq; ++i) {
            const int st = i % kQDStages;
            mbar_wait(&qd_full[st], (i / kQDStages) & 1);
            BWD_TRACE(i, 5);
            if (i >= 1) mbar_wait(s_free, (i - 1) & 1);
            BWD_TRACE(i, 0);
            tc_fence_after();
            uint8_t *qdst = smem + kB_QD + st * 2 * kTileBytes;
            const uint64_t qk = sdesc_sw(smem_u32(qdst), 1024, 2);
            const uint64_t dok = sdesc_sw(smem_u32(qdst + kTileBytes), 1024, 2);
#pragma unroll
            for (int k = 0; k < kD / 16; ++k) {
                if (p.dbg & 8) break;
                mma_bf16_e(tmem + kColST, kd + ((k * 32) >> 4), qk + ((k * 32) >> 4), id_s,
                           k ? 1u : 0u);
                mma_bf16_e(tmem + kColDP, vd + ((k * 32) >> 4), dok + ((k * 32) >> 4), id_s,
                           k ? 1u : 0u);
            }
            mma_commit_e(s_full);
            BWD_TRACE(i, 15);
            if (i >= 1) issue_grads(i - 1);
        }
        if (nq >= 1) issue_grads(nq - 1);
    }
    } else if (warp < 20) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 88;");
        // ============ P^T / dS^T (thread = key row, 32-column quarter) ============
        const int quarter = warp & 3;
        const int cq = (warp - 4) >> 2;                  // query columns [32 cq, 32 cq + 32)
        const int rl = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const float2 c2 = make_float2(p.c, p.c);
        const float2 sc2 = make_float2(p.scale, p.scale);
        for (int i = 0; i < nq; ++i) {
            const int b = i & 1;
            const int lb = i % kLDBufs;
            mbar_wait(&ld_full[lb], (i / kLDBufs) & 1);   // this block's -LSE2 / D rows staged
            mbar_wait(s_full, i & 1);
            if (warp == 4) BWD_TRACE(i, 4);
            tc_fence_after();
            uint8_t *ps = smem + kB_PS + b * kPBytes + rl * 128 + (cq >> 1) * (kBN * 128);   // dS^T(b)
            const float *NL2 = lse2_s + lb * 128 + cq * 32;
            const float *Dl = delta_s + lb * 128 + cq * 32;
            uint32_t pall[16];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {          // 16 query columns at a time
                uint32_t sv[16], dv[16];
                const uint32_t col = cq * 32 + cc * 16;
                tmem_ld16(lane_base + kColST + col, sv);
                tmem_ld16(lane_base + kColDP + col, dv);
                tmem_wait_ld();
                if (cc == 1) {
                    tc_fence_before();
                    mbar_arrive(s_free);   // S^T / dP^T TMEM may be overwritten
                    if (warp == 4) BWD_TRACE(i, 6);
                } else {
                    if (i >= 2) mbar_wait(&ds_empty[b], ((i - 2) >> 1) & 1);   // dS^T(b) free
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {         // 16-B chunks of 8 query columns
                    if (p.dbg & 2) break;
                    uint32_t dk4[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int qc = c * 8 + 2 * e;
                        const float2 nl = *reinterpret_cast<const float2 *>(NL2 + cc * 16 + qc);
                        const float2 dd = *reinterpret_cast<const float2 *>(Dl + cc * 16 + qc);
                        float2 x = ffma2(make_float2(__uint_as_float(sv[qc]), __uint_as_float(sv[qc + 1])),
                                         c2, nl);
                        x.x = ex2(x.x);
                        x.y = ex2(x.y);
                        const float2 g = fmul2(
                            x, ffma2(make_float2(__uint_as_float(dv[qc]), __uint_as_float(dv[qc + 1])),
                                     sc2, make_float2(-dd.x, -dd.y)));
                        pall[cc * 8 + c * 4 + e] = pack_bf16(x.x, x.y);
                        dk4[e] = pack_bf16(g.x, g.y);
                    }
                    const int chunk = (cq & 1) * 4 + cc * 2 + c;   // 16-B chunk in the 128-B half-tile row
                    *reinterpret_cast<uint4 *>(ps + ((chunk ^ (rl & 7)) << 4)) =
                        make_uint4(dk4[0], dk4[1], dk4[2], dk4[3]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ld_empty[lb]);     // done reading the staged rows
            // P^T pairs (q, q+1) -> TMEM column kColPT + q / 2 (the TS A layout).
            // Written last: dV(i-1), issued when block i-1's softmax finished,
            // has had this whole block's softmax math to read the previous P^T.
            if (warp == 4) BWD_TRACE(i, 7);
            if (i >= 1 && !(p.dbg & 64)) mbar_wait(pv_empty, (i - 1) & 1);
            if (warp == 4) BWD_TRACE(i, 9);
            tc_fence_after();
            if (!(p.dbg & 2)) tmem_st16(lane_base + kColPT + cq * 16, pall);
            tmem_wait_st();
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(&p_full[b]);
            if (warp == 4) BWD_TRACE(i, 10);
        }
        // dV (cq 0, 1) / dK (cq 2, 3) 32-column halves += TMEM once the last
        // gradient MMAs have landed
        if (nq >= 1) mbar_wait(&ds_empty[(nq - 1) & 1], ((nq - 1) >> 1) & 1);
        tc_fence_after();
        const int key = k0 + rl;
        const bool kv_ok = key < p.sk;
        const size_t ki = ((size_t)key * p.H + h) * kD;
        float *gdst = cq >= 2 ? p.dk : p.dv;
        const int c0 = (cq & 1) * 32;
        const uint32_t gcol = (cq >= 2 ? kColDK : kColDV) + c0;
        for (int c = 0; c < 32; c += 16) {
            uint32_t a[16];
            tmem_ld16(lane_base + gcol + c, a);
            tmem_wait_ld();
            if (kv_ok) {
                float4 *pv = reinterpret_cast<float4 *>(gdst + ki + c0 + c);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float4 x = pv[e];
                    x.x += __uint_as_float(a[4 * e]); x.y += __uint_as_float(a[4 * e + 1]);
                    x.z += __uint_as_float(a[4 * e + 2]); x.w += __uint_as_float(a[4 * e + 3]);
                    pv[e] = x;
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
        // ===================== dQ epilogue (thread = query row) =====================
        const int quarter = warp & 3;
        const int rl = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const bool leader = warp == 20;
        // -LSE*log2(e) and scale*D of query block q -> ring slot q % kLDBufs
        // (strided global loads, off the softmax's critical path).  The loads
        // for block i + 3 are issued right after block i + 2's rows are
        // stored, so their latency overlaps this warp's dQ wait and drain.
        float l_pf = INFINITY, d_pf = 0.f;
        auto fetch_rows = [&](int q) {
            l_pf = INFINITY;
            d_pf = 0.f;
            const int qrow = q * kBM + rl;
            if (q < nq && qrow < p.sq) {
                const size_t qi = (size_t)qrow * p.H + h;
                l_pf = __ldg(p.lse + qi);
                d_pf = __ldg(p.delta + qi);
            }
        };
        auto store_rows = [&](int q) {
            if (q >= nq) return;
            const int sl = q % kLDBufs;
            if (q >= kLDBufs) mbar_wait(&ld_empty[sl], ((q / kLDBufs) - 1) & 1);
            lse2_s[sl * 128 + rl] = -l_pf * kLog2e;
            delta_s[sl * 128 + rl] = d_pf * p.scale;   // dS = P (scale dP - scale D)
            mbar_arrive(&ld_full[sl]);
        };
        fetch_rows(0);
        store_rows(0);
        fetch_rows(1);
        store_rows(1);
        fetch_rows(2);
        for (int i = 0; i < nq; ++i) {
            store_rows(i + 2);
            fetch_rows(i + 3);
            mbar_wait(dq_full, i & 1);
            if (warp == 20) BWD_TRACE(i, 12);
            tc_fence_after();
            // the staging tile was last reduced one block ago: its TMA reads must be done
            if (leader && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            named_bar(2, 128);
            uint8_t *stg = smem + kB_DQ;
            for (int c = 0; c < kD; c += 16) {
                uint32_t a[16];
                tmem_ld16(lane_base + kColDQ + c, a);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int chunk = (c >> 2) + e;              // 16-B chunk of 4 floats, 0..15
                    const int hf = chunk >> 3, cc = chunk & 7;   // 32-column box, chunk in row
                    *reinterpret_cast<uint4 *>(stg + hf * (kDQStage / 2) + rl * 128 +
                                               ((cc ^ (rl & 7)) << 4)) =
                        make_uint4(a[4 * e], a[4 * e + 1], a[4 * e + 2], a[4 * e + 3]);
                }
            }
            tc_fence_before();
            mbar_arrive(dq_empty);            // TMEM dQ free
            if (warp == 20) BWD_TRACE(i, 13);
            fence_async_smem();
            named_bar(2, 128);
            if (leader) {
                if (lane == 0 && !(p.dbg & 1)) {
                    for (int hf = 0; hf < 2; ++hf)
                        asm volatile(
                            "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group "
                            "[%0, {%1, %2, %3}], [%4];" ::"l"(reinterpret_cast<uint64_t>(&dqmap)),
                            "r"(hf * 32), "r"(h), "r"(i * kBM),
                            "r"(smem_u32(stg + hf * (kDQStage / 2)))
                            : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                __syncwarp();
            }
        }
        if (leader && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// [S, H, 64] bf16 view with element strides (row, head): box 64 x 1 x 128,
// 128-B swizzle.
int head_map(CUtensorMap *m, const void *base, int64_t rows, int64_t heads, int64_t rs, int64_t hs) {
    uint64_t dims[3] = {(uint64_t)kD, (uint64_t)heads, (uint64_t)rows};
    uint64_t strides[2] = {(uint64_t)hs * 2, (uint64_t)rs * 2};
    uint32_t box[3] = {(uint32_t)kD, 1, (uint32_t)kBM};
    return encode_tensor_map(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims,
                             strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace

int attn_tc_eligible(const dp_attn_geom *g, int dtype) {
    if (!g || dtype != DP_BF16 || g->dim != kD) return 0;
    const int64_t s[6] = {g->q_rs, g->q_hs, g->k_rs, g->k_hs, g->v_rs, g->v_hs};
    for (int i = 0; i < 6; ++i)
        if (s[i] % 8) return 0;  // 16-B aligned TMA strides
    if (g->sq > (1 << 30) || g->sk > (1 << 30)) return 0;
    return 1;
}

int attn_fwd_update_tc_launch(const dp_attn_geom *g, const void *q, const void *k, const void *v,
                              void *m, void *l, void *acc, cudaStream_t st) {
    DP_REQUIRE(attn_tc_eligible(g, DP_BF16), DP_ERR_UNSUPPORTED, "attn_tc: outside the envelope");
    if (g->sq == 0 || g->sk == 0) return DP_OK;
    CUtensorMap qm, km, vm;
    int rc = head_map(&qm, q, g->sq, g->heads, g->q_rs, g->q_hs);
    if (!rc) rc = head_map(&km, k, g->sk, g->heads, g->k_rs, g->k_hs);
    if (!rc) rc = head_map(&vm, v, g->sk, g->heads, g->v_rs, g->v_hs);
    if (rc) return rc;
    FwdParams p;
    p.sq = (int)g->sq;
    p.sk = (int)g->sk;
    p.H = (int)g->heads;
    p.n_qt = (int)((g->sq + kBM * kFwdTiles - 1) / (kBM * kFwdTiles));
    p.c = (float)(g->scale * 1.4426950408889634);
    p.m = (float *)m;
    p.l = (float *)l;
    p.acc = (float *)acc;
    static int poly = -1;  // DP_ATTN_POLY: exp2 pairs per 8 on the FMA pipe (tuning knob)
    if (poly < 0) {
        const char *e = getenv("DP_ATTN_POLY");
        poly = e ? atoi(e) : 2;
        if (poly < 0 || poly > 4) poly = 2;
    }
    auto kern = poly == 0 ? attn_fwd_tc_kernel<0> : poly == 1 ? attn_fwd_tc_kernel<1>
              : poly == 2 ? attn_fwd_tc_kernel<2> : poly == 3 ? attn_fwd_tc_kernel<3>
                                                  : attn_fwd_tc_kernel<4>;
    DP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFwd));
    const int64_t grid = (int64_t)p.n_qt * p.H;
    kern<<<(unsigned)grid, kFwdThreads, kSmemFwd, st>>>(qm, km, vm, p);
    return launch_status("attn_fwd_tc_kernel");
}

int attn_bwd_tc_eligible(const dp_attn_geom *g, int dtype) {
    if (!attn_tc_eligible(g, dtype)) return 0;
    return (g->o_rs % 8 == 0 && g->o_hs % 8 == 0) ? 1 : 0;
}

int attn_bwd_update_tc_launch(const dp_attn_geom *g, const void *q, const void *k, const void *v,
                              const void *dout, const void *lse, const void *delta, void *dq,
                              void *dk, void *dv, cudaStream_t st) {
    DP_REQUIRE(attn_bwd_tc_eligible(g, DP_BF16), DP_ERR_UNSUPPORTED,
               "attn_tc bwd: outside the envelope");
    if (g->sq == 0 || g->sk == 0) return DP_OK;
    CUtensorMap qm, km, vm, dm;
    int rc = head_map(&qm, q, g->sq, g->heads, g->q_rs, g->q_hs);
    if (!rc) rc = head_map(&km, k, g->sk, g->heads, g->k_rs, g->k_hs);
    if (!rc) rc = head_map(&vm, v, g->sk, g->heads, g->v_rs, g->v_hs);
    if (!rc) rc = head_map(&dm, dout, g->sq, g->heads, g->o_rs, g->o_hs);
    CUtensorMap dqm;  // dq [sq, H, 64] fp32, box 32 x 1 x 128 (128-B swizzle): reduce-add target
    if (!rc) {
        uint64_t dims[3] = {(uint64_t)kD, (uint64_t)g->heads, (uint64_t)g->sq};
        uint64_t strides[2] = {(uint64_t)kD * 4, (uint64_t)g->heads * kD * 4};
        uint32_t box[3] = {32, 1, (uint32_t)kBM};
        rc = encode_tensor_map(&dqm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dq, dims, strides, box,
                               CU_TENSOR_MAP_SWIZZLE_128B);
    }
    if (rc) return rc;
    BwdParams p;
    p.sq = (int)g->sq;
    p.sk = (int)g->sk;
    p.H = (int)g->heads;
    p.n_kt = (int)((g->sk + kBN - 1) / kBN);
    p.c = (float)(g->scale * 1.4426950408889634);
    p.scale = (float)g->scale;
    p.lse = (const float *)lse;
    p.delta = (const float *)delta;
    p.dq = (float *)dq;
    p.dk = (float *)dk;
    p.dv = (float *)dv;
    {
        static int dbg = -1;
        if (dbg < 0) {
            const char *e = getenv("DP_ATTN_DBG");
            dbg = e ? atoi(e) : 0;
        }
        p.dbg = dbg;
    }
    static unsigned long long *trace = nullptr;
    static int want_trace = -1;
    if (want_trace < 0) want_trace = getenv("DP_ATTN_TRACE") ? 1 : 0;
    if (want_trace && !trace) DP_CUDA_CHECK(cudaMalloc(&trace, 64 * 16 * 8));
    if (trace) DP_CUDA_CHECK(cudaMemsetAsync(trace, 0, 64 * 16 * 8, st));
    p.trace = trace;
    DP_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBwd));
    const int64_t grid = (int64_t)p.n_kt * p.H;
    attn_bwd_tc_kernel<<<(unsigned)grid, kBwdThreads, kSmemBwd, st>>>(qm, km, vm, dm, dqm, p);
    if (trace) {  // debug: CTA 0's per-block event clocks relative to block 20's s_full
        unsigned long long hbuf[64 * 16];
        DP_CUDA_CHECK(cudaStreamSynchronize(st));
        DP_CUDA_CHECK(cudaMemcpy(hbuf, trace, sizeof hbuf, cudaMemcpyDeviceToHost));
        const long long t0 = (long long)hbuf[20 * 16 + 4];
        fprintf(stderr, "blk  Msfree  Mpful  Mdqem   MdV  Ssful  Mqdfl  Ssfre  Smath  MdVdK  Spvem  Spful  Mgrds  Qdqfl  Qdrn  Pqdem  Mscmt\n");
        for (int bb = 18; bb < 26; ++bb) {
            fprintf(stderr, "%3d", bb);
            for (int e = 0; e < 16; ++e)
                fprintf(stderr, " %6lld", hbuf[bb * 16 + e] ? (long long)hbuf[bb * 16 + e] - t0 : -1);
            fprintf(stderr, "\n");
        }
    }
    return launch_status("attn_bwd_tc_kernel");
}

}  // namespace dp
