// fp32 convolution on the bf16 tensor cores, fp32-accurate ("bf16x3").
//
// The reference computes conv in fp32/fp64 and holds fp32 to 1e-5
// (domainpar/verify.py:40), which rules out plain bf16 or TF32 tensor math.
// Every fp32 value splits exactly into three bf16 parts, x = xh + xm + xl
// (8 + 8 + 8 significand bits >= fp32's 24), and the product of two fp32
// values is, to ~2^-24 relative, the six leading part products
//     xh wh + xh wm + xh wl + xm wh + xm wm + xl wh.
// Those six terms become ONE bf16 convolution with fp32 accumulation in TMEM
// by concatenating along the contraction:
//   fwd    channels: X' = [xh xh xh xm xm xl] (6 C_in), W' = [wh wm wl wh wm wh]
//          (X' is virtual: the operand stores [xh xm xl] once and the conv
//          kernel's K block b reads part c_xpat[b] — conv_tc.cu X3)
//   dgrad  channels: dY' = [dh dh dh dm dm dl] (6 C_out), W' split on c_out
//   wgrad  batch:    pairs (xh dh, xm dh, xh dm, xl dh, xm dm, xh dl)
// (wgrad contracts over positions, so the six pairings are six batch entries
// of a bf16 wgrad whose batch sum is the answer; X and dY hold their 3 parts
// once as batch blocks and the TS wgrad kernel maps batch entry k to its
// (X part, dY part) pair, conv_tc.cu kTsPairX / kTsPairD).  Split kernels write the
// channels-last bf16 operands (a tiled transpose from the caller's fp32
// strides); the tcgen05 kernels of conv_tc.cu run unchanged except for an
// fp32-output epilogue.  Measured error vs fp64: ~1e-7 (tests/).
#include "common.cuh"

namespace dp {

int64_t conv_tc_f32out_workspace(const dp_conv_geom *g, bool dgrad);
int conv_tc_f32out_launch(const dp_conv_geom *g, bool dgrad, const void *in, const void *in_halo,
                          const void *w, void *out, void *out2, void *ws, int64_t ws_bytes,
                          cudaStream_t st);
int conv_wgrad_x3_launch(const dp_conv_geom *g, const void *x, const void *xh, const void *dy,
                         void *dw, void *ws, int64_t ws_bytes, cudaStream_t st, int B);
int64_t conv_wgrad_x3_workspace(const dp_conv_geom *g);
int conv_tc_eligible(const dp_conv_geom *g, int dtype, int which);
int64_t conv_tc_workspace(const dp_conv_geom *g, int which);
int conv_wgrad_tc_launch(const dp_conv_geom *g, const void *x, const void *xh, const void *dy,
                         void *dw, void *ws, int64_t ws_bytes, cudaStream_t st);

namespace {

constexpr int kParts = 6;
// part index (0 = hi, 1 = mid, 2 = lo) of each concatenated block
__constant__ int c_xpat[kParts] = {0, 0, 0, 1, 1, 2};   // activations (fwd / dgrad input)
__constant__ int c_wpat[kParts] = {0, 1, 2, 0, 1, 0};   // weights
__constant__ int c_ppat[kParts] = {0, 1, 0, 2, 1, 0};   // wgrad X'' (6 blocks, SS fallback)
__constant__ int c_dpat[kParts] = {0, 0, 1, 0, 1, 2};   // wgrad dY'' (6 blocks, SS fallback)
__constant__ int c_ipat[kParts] = {0, 1, 2, 0, 0, 0};   // the 3 parts once (wgrad, paired
                                                        // in the kernel: conv_tc.cu kTsPair*)

__device__ __forceinline__ void split3(float x, __nv_bfloat16 (&pt)[3]) {
    pt[0] = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(pt[0]);
    pt[1] = __float2bfloat16_rn(r1);
    pt[2] = __float2bfloat16_rn(r1 - __bfloat162float(pt[1]));
}

// fp32 activation [B][C][S0][S1] (any strides, 2-D) -> bf16 channels-last.
// mode 0: channel blocks out[b][s0][s1][blk*C + c] = part_{pat[blk]} (nblk blocks);
// mode 1: batch blocks out[blk*B + b][s0][s1][c] = part_{pat[blk]}.
// Tile: 32 channels x 64 positions along S1 through smem — coalesced fp32
// reads along S1; then a thread splits 8 consecutive channels of one
// position and writes each part as one 16-B vector (C % 8 == 0).
__global__ void __launch_bounds__(256)
x3_split_act(const float *__restrict__ x, int64_t B, int64_t C, int64_t S0, int64_t S1,
             int64_t sb, int64_t sc, int64_t s0, int64_t s1, __nv_bfloat16 *__restrict__ out,
             int mode, int which_pat) {
    __shared__ float tile[32][65];
    const int *pat = which_pat == 0 ? c_xpat : which_pat == 1 ? c_ipat
                     : which_pat == 2 ? c_ppat : c_dpat;
    const int nblk = which_pat == 1 ? 3 : kParts;
    const int64_t n1 = (S1 + 63) / 64, nc = (C + 31) / 32;
    int64_t t = blockIdx.x;
    const int64_t t1 = t % n1; t /= n1;
    const int64_t tc = t % nc; t /= nc;
    const int64_t i0 = t % S0;
    const int64_t b = t / S0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const float *src = x + b * sb + i0 * s0;
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = tc * 32 + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t i1 = t1 * 64 + h * 32 + tx;
            tile[k][h * 32 + tx] = (c < C && i1 < S1) ? src[c * sc + i1 * s1] : 0.f;
        }
    }
    __syncthreads();
    const int pos = threadIdx.x >> 2, cg = threadIdx.x & 3;   // 64 positions x 4 groups of 8
    const int64_t i1 = t1 * 64 + pos, c0 = tc * 32 + cg * 8;
    if (i1 >= S1 || c0 >= C) return;
    uint32_t pk[3][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        __nv_bfloat16 a[3], bb[3];
        split3(tile[cg * 8 + 2 * e][pos], a);
        split3(tile[cg * 8 + 2 * e + 1][pos], bb);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            __nv_bfloat162 v;
            v.x = a[q];
            v.y = bb[q];
            pk[q][e] = *reinterpret_cast<uint32_t *>(&v);
        }
    }
#pragma unroll
    for (int blk = 0; blk < kParts; ++blk) {
        if (blk >= nblk) break;
        const int q = pat[blk];
        const uint4 v = make_uint4(pk[q][0], pk[q][1], pk[q][2], pk[q][3]);
        __nv_bfloat16 *dst =
            mode == 0 ? out + ((b * S0 + i0) * S1 + i1) * (nblk * C) + blk * C + c0
                      : out + ((((int64_t)blk * B + b) * S0 + i0) * S1 + i1) * C + c0;
        *reinterpret_cast<uint4 *>(dst) = v;
    }
}

// fp32 weights [Co][Ci][T] -> bf16: mode 0 (fwd)   W'[co][blk*Ci + ci][t]
//                                   mode 1 (dgrad) W'[blk*Co + co][ci][t]
__global__ void x3_split_weight(const float *__restrict__ w, int64_t Co, int64_t Ci, int64_t T,
                                __nv_bfloat16 *__restrict__ out, int mode) {
    const int64_t n = Co * Ci * T;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e % T, ci = (e / T) % Ci, co = e / (T * Ci);
        __nv_bfloat16 pt[3];
        split3(w[e], pt);
#pragma unroll
        for (int blk = 0; blk < kParts; ++blk) {
            const int64_t idx = mode == 0 ? (co * (kParts * Ci) + blk * Ci + ci) * T + t
                                          : (((int64_t)blk * Co + co) * Ci + ci) * T + t;
            out[idx] = pt[c_wpat[blk]];
        }
    }
}

struct X3Layout {
    int64_t act, act_h, wimg, dy, dy_h, inner, total;   // byte offsets / sizes
};

int64_t align256(int64_t v) { return (v + 255) & ~int64_t(255); }

// channels-last contiguous strides [b, c, s0, s1] of a [B][S0][S1][C] tensor
void cl_strides(int64_t S0, int64_t S1, int64_t C, int64_t *s) {
    s[0] = S0 * S1 * C;
    s[1] = 1;
    s[2] = S1 * C;
    s[3] = C;
    s[4] = 0;
}

bool x3_shape_ok(const dp_conv_geom *g) {
    if (g->nsp != 2 || g->kernel[0] != 3 || g->kernel[1] != 3) return false;
    if (g->stride[0] != 1 || g->stride[1] != 1) return false;
    if (!(g->c_in == 16 || g->c_in == 32) || !(g->c_out == 16 || g->c_out == 32)) return false;
    if (!(g->shard == -1 || g->shard == 0)) return false;
    return true;
}

// geometry of the bf16 conv over the split operands
dp_conv_geom x3_geom(const dp_conv_geom *g, int which) {
    dp_conv_geom h = *g;
    const int64_t Hin = g->in_ext[0], Win = g->in_ext[1];
    const int64_t Hout = g->out_ext[0], Wout = g->out_ext[1];
    // fwd / dgrad: the MMA contracts over 6 C channel blocks, the stored operand
    // holds the 3 parts once (3 C channels; conv_tc.cu X3)
    if (which == DP_CONV_FWD) {
        h.c_in = kParts * g->c_in;
        cl_strides(Hin, Win, 3 * g->c_in, h.xs);
        cl_strides(g->halo, Win, 3 * g->c_in, h.hs);
    } else if (which == DP_CONV_DGRAD) {
        h.c_out = kParts * g->c_out;
        cl_strides(Hout, Wout, 3 * g->c_out, h.ys);
    } else {
        h.batch = kParts * g->batch;
        cl_strides(Hin, Win, g->c_in, h.xs);
        cl_strides(g->halo, Win, g->c_in, h.hs);
        cl_strides(Hout, Wout, g->c_out, h.ys);
    }
    return h;
}

// the TS wgrad kernel pairs the parts itself (3 + 3 parts); other shapes run
// the SS wgrad kernel over the 6 materialised pairings
bool x3_wgrad_paired(const dp_conv_geom *g) {
    const dp_conv_geom h = x3_geom(g, DP_CONV_WGRAD);
    return conv_wgrad_x3_workspace(&h) >= 0;
}

X3Layout x3_layout(const dp_conv_geom *g, int which) {
    X3Layout L{};
    const int64_t Hin = g->in_ext[0], Win = g->in_ext[1];
    const int64_t Hout = g->out_ext[0], Wout = g->out_ext[1];
    const int64_t taps = 9;
    int64_t off = 0;
    if (which == DP_CONV_FWD) {
        L.act = off; off += align256(g->batch * Hin * Win * 3 * g->c_in * 2);
        L.act_h = off; off += align256(g->batch * g->halo * Win * 3 * g->c_in * 2);
        L.wimg = off; off += align256(g->c_out * kParts * g->c_in * taps * 2);
    } else if (which == DP_CONV_DGRAD) {
        L.dy = off; off += align256(g->batch * Hout * Wout * 3 * g->c_out * 2);
        L.wimg = off; off += align256(kParts * g->c_out * g->c_in * taps * 2);
    } else {
        const int64_t np = x3_wgrad_paired(g) ? 3 : kParts;   // parts once, or 6 pairings
        L.act = off; off += align256(np * g->batch * Hin * Win * g->c_in * 2);
        L.act_h = off; off += align256(np * g->batch * g->halo * Win * g->c_in * 2);
        L.dy = off; off += align256(np * g->batch * Hout * Wout * g->c_out * 2);
    }
    L.inner = off;
    const dp_conv_geom h = x3_geom(g, which);
    const int64_t in_ws = which != DP_CONV_WGRAD
                              ? conv_tc_f32out_workspace(&h, which == DP_CONV_DGRAD)
                              : (x3_wgrad_paired(g) ? conv_wgrad_x3_workspace(&h)
                                                    : conv_tc_workspace(&h, DP_CONV_WGRAD));
    L.total = in_ws < 0 ? -1 : off + align256(in_ws);
    return L;
}

int launch_split(const float *x, int64_t B, int64_t C, int64_t S0, int64_t S1, const int64_t *st,
                 __nv_bfloat16 *out, int mode, int pat, cudaStream_t s) {
    if (B * C * S0 * S1 == 0) return DP_OK;
    const int64_t blocks = B * S0 * ((C + 31) / 32) * ((S1 + 63) / 64);
    DP_REQUIRE(blocks < (1ll << 31), DP_ERR_UNSUPPORTED, "x3 split: grid too large");
    x3_split_act<<<(unsigned)blocks, 256, 0, s>>>(x, B, C, S0, S1, st[0], st[1], st[2], st[3], out,
                                                  mode, pat);
    return launch_status("x3_split_act");
}

}  // namespace

int conv_x3_eligible(const dp_conv_geom *g, int which) {
    if (!g || !x3_shape_ok(g)) return 0;
    if (which == DP_CONV_WGRAD) {
        const dp_conv_geom h = x3_geom(g, which);
        return (conv_wgrad_x3_workspace(&h) >= 0 || conv_tc_eligible(&h, DP_BF16, DP_CONV_WGRAD))
                   ? 1 : 0;
    }
    const dp_conv_geom h = x3_geom(g, which);
    return conv_tc_f32out_workspace(&h, which == DP_CONV_DGRAD) >= 0 ? 1 : 0;
}

int64_t conv_x3_workspace(const dp_conv_geom *g, int which) {
    if (!conv_x3_eligible(g, which)) return -1;
    return x3_layout(g, which).total;
}

int conv_x3_launch(const dp_conv_geom *g, int which, const void *a, const void *ah, const void *b,
                   void *out, void *out2, void *ws, int64_t ws_bytes, cudaStream_t st) {
    DP_REQUIRE(conv_x3_eligible(g, which), DP_ERR_UNSUPPORTED, "conv_x3: outside the envelope");
    const X3Layout L = x3_layout(g, which);
    DP_REQUIRE(L.total >= 0 && ws_bytes >= L.total, DP_ERR_INVALID, "conv_x3: workspace too small");
    uint8_t *w8 = (uint8_t *)ws;
    const dp_conv_geom h = x3_geom(g, which);
    const int64_t Hin = g->in_ext[0], Win = g->in_ext[1];
    const int64_t Hout = g->out_ext[0], Wout = g->out_ext[1];
    int rc;
    if (which == DP_CONV_FWD) {            // a = x, ah = x halo, b = w (fp32), out = y
        __nv_bfloat16 *xa = (__nv_bfloat16 *)(w8 + L.act), *xha = (__nv_bfloat16 *)(w8 + L.act_h);
        __nv_bfloat16 *wi = (__nv_bfloat16 *)(w8 + L.wimg);
        int64_t sx[4] = {g->xs[0], g->xs[1], g->xs[2], g->xs[3]};
        if ((rc = launch_split((const float *)a, g->batch, g->c_in, Hin, Win, sx, xa, 0, 1, st)))
            return rc;
        if (g->halo > 0) {
            int64_t sh[4] = {g->hs[0], g->hs[1], g->hs[2], g->hs[3]};
            if ((rc = launch_split((const float *)ah, g->batch, g->c_in, g->halo, Win, sh, xha, 0, 1,
                                   st)))
                return rc;
        }
        const int64_t nw = g->c_out * g->c_in * 9;
        x3_split_weight<<<grid_for(nw, 256, 2), 256, 0, st>>>((const float *)b, g->c_out, g->c_in, 9,
                                                              wi, 0);
        if ((rc = launch_status("x3_split_weight"))) return rc;
        return conv_tc_f32out_launch(&h, false, xa, g->halo > 0 ? xha : nullptr, wi, out, nullptr,
                                     w8 + L.inner, ws_bytes - L.inner, st);
    }
    if (which == DP_CONV_DGRAD) {          // a = dy, b = w (fp32), out = dx, out2 = dx halo
        __nv_bfloat16 *da = (__nv_bfloat16 *)(w8 + L.dy), *wi = (__nv_bfloat16 *)(w8 + L.wimg);
        int64_t sd[4] = {g->ys[0], g->ys[1], g->ys[2], g->ys[3]};
        if ((rc = launch_split((const float *)a, g->batch, g->c_out, Hout, Wout, sd, da, 0, 1, st)))
            return rc;
        const int64_t nw = g->c_out * g->c_in * 9;
        x3_split_weight<<<grid_for(nw, 256, 2), 256, 0, st>>>((const float *)b, g->c_out, g->c_in, 9,
                                                              wi, 1);
        if ((rc = launch_status("x3_split_weight"))) return rc;
        return conv_tc_f32out_launch(&h, true, da, nullptr, wi, out, out2, w8 + L.inner,
                                     ws_bytes - L.inner, st);
    }
    // wgrad: a = x, ah = x halo, b = dy, out = dw (fp32)
    __nv_bfloat16 *xa = (__nv_bfloat16 *)(w8 + L.act), *xha = (__nv_bfloat16 *)(w8 + L.act_h);
    __nv_bfloat16 *da = (__nv_bfloat16 *)(w8 + L.dy);
    const bool paired = x3_wgrad_paired(g);
    const int px = paired ? 1 : 2, pd = paired ? 1 : 3;
    int64_t sx[4] = {g->xs[0], g->xs[1], g->xs[2], g->xs[3]};
    if ((rc = launch_split((const float *)a, g->batch, g->c_in, Hin, Win, sx, xa, 1, px, st)))
        return rc;
    if (g->halo > 0) {
        int64_t sh[4] = {g->hs[0], g->hs[1], g->hs[2], g->hs[3]};
        if ((rc = launch_split((const float *)ah, g->batch, g->c_in, g->halo, Win, sh, xha, 1, px,
                               st)))
            return rc;
    }
    int64_t sd[4] = {g->ys[0], g->ys[1], g->ys[2], g->ys[3]};
    if ((rc = launch_split((const float *)b, g->batch, g->c_out, Hout, Wout, sd, da, 1, pd, st)))
        return rc;
    if (!paired)
        return conv_wgrad_tc_launch(&h, xa, g->halo > 0 ? xha : nullptr, da, out, w8 + L.inner,
                                    ws_bytes - L.inner, st);
    return conv_wgrad_x3_launch(&h, xa, g->halo > 0 ? xha : nullptr, da, out, w8 + L.inner,
                                ws_bytes - L.inner, st, (int)g->batch);
}

}  // namespace dp
