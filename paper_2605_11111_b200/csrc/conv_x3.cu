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
//          (X' is virtual: the operand stores [xh xm xl] once, as batch
//          blocks, and the conv kernel's K block b reads part c_xpat[b] —
//          conv_tc.cu X3; the same split operands feed the wgrad, so the
//          host splits x once in the forward and dy once in the backward:
//          dp_conv_x3_split + dp_conv_x3_*_parts, ops.py keeps x's parts
//          in the conv tape)
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
                     : c_xpat;
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

// The split of a dense fp32 NCHW-like operand (unit S1 stride, 16-B aligned
// rows, S1 % 128 == 0) into the 3 parts as batch blocks out[part*B + b]
// [s0][s1][c]: a block moves 32 channels x 128 positions — float4 reads (one
// 512-B channel row per warp instruction) into a column-swizzled smem tile
// (column ^= 8 * channel group: conflict-free reads of 8 channels at one
// position), then thread (position, channel group of 8) splits its 8
// channels and writes each part as 16 B; a warp writes 8 positions x 4
// groups = contiguous 512-B runs (C = 32).  ~1.3x the scalar tile kernel.
__global__ void __launch_bounds__(256)
x3_split_act_v4(const float *__restrict__ x, int64_t B, int64_t C, int64_t S0, int64_t S1,
                int64_t sb, int64_t sc, int64_t s0, __nv_bfloat16 *__restrict__ out) {
    __shared__ __align__(16) float tile[32][132];
    const int64_t n1 = S1 / 128, nc = (C + 31) / 32;
    int64_t t = blockIdx.x;
    const int64_t t1 = t % n1; t /= n1;
    const int64_t tc = t % nc; t /= nc;
    const int64_t i0 = t % S0;
    const int64_t b = t / S0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float *src = x + b * sb + i0 * s0 + t1 * 128;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int c = warp * 4 + r;
        if (tc * 32 + c < C) {
            const float4 v = *reinterpret_cast<const float4 *>(src + (tc * 32 + c) * sc + lane * 4);
            *reinterpret_cast<float4 *>(&tile[c][(lane * 4) ^ ((c >> 3) << 3)]) = v;
        }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int it = threadIdx.x + 256 * h;
        const int pos = it >> 2, cg = it & 3;
        const int64_t c0 = tc * 32 + cg * 8;
        if (c0 >= C) continue;
        uint32_t pk[3][4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            __nv_bfloat16 a[3], bb[3];
            split3(tile[cg * 8 + 2 * e][pos ^ (cg << 3)], a);
            split3(tile[cg * 8 + 2 * e + 1][pos ^ (cg << 3)], bb);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                __nv_bfloat162 v;
                v.x = a[q];
                v.y = bb[q];
                pk[q][e] = *reinterpret_cast<uint32_t *>(&v);
            }
        }
        const int64_t i1 = t1 * 128 + pos;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            __nv_bfloat16 *dst = out + ((((int64_t)q * B + b) * S0 + i0) * S1 + i1) * C + c0;
            *reinterpret_cast<uint4 *>(dst) = make_uint4(pk[q][0], pk[q][1], pk[q][2], pk[q][3]);
        }
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

// Geometry of the bf16 conv over the split operands.  Every split operand is
// the 3 parts once as batch blocks [3][B][S0][S1][C] channels-last (strides
// of one [B][..][C] block here); fwd / dgrad contract over the virtual 6 C
// channel blocks (conv_tc.cu X3), wgrad pairs the parts as 6 batch entries.
dp_conv_geom x3_geom(const dp_conv_geom *g, int which) {
    dp_conv_geom h = *g;
    const int64_t Hin = g->in_ext[0], Win = g->in_ext[1];
    const int64_t Hout = g->out_ext[0], Wout = g->out_ext[1];
    if (which == DP_CONV_FWD) {
        h.c_in = kParts * g->c_in;
        cl_strides(Hin, Win, g->c_in, h.xs);
        cl_strides(g->halo, Win, g->c_in, h.hs);
    } else if (which == DP_CONV_DGRAD) {
        h.c_out = kParts * g->c_out;
        cl_strides(Hout, Wout, g->c_out, h.ys);
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

// bytes of one split operand (DP_X3_X: x main block, DP_X3_XHALO: the
// received x halo rows, DP_X3_DY: dy), 3 parts
int64_t x3_operand_bytes(const dp_conv_geom *g, int operand) {
    const int64_t Win = g->in_ext[1];
    if (operand == DP_X3_X) return 3 * g->batch * g->in_ext[0] * Win * g->c_in * 2;
    if (operand == DP_X3_XHALO) return 3 * g->batch * g->halo * Win * g->c_in * 2;
    if (operand == DP_X3_DY) return 3 * g->batch * g->out_ext[0] * g->out_ext[1] * g->c_out * 2;
    return -1;
}

// workspace of a launch over already-split operands: the weight image (fwd /
// dgrad) + the tcgen05 kernel's own workspace
int64_t x3_inner_bytes(const dp_conv_geom *g, int which, int64_t *wimg_bytes) {
    const dp_conv_geom h = x3_geom(g, which);
    int64_t wimg = 0;
    int64_t in_ws;
    if (which == DP_CONV_WGRAD) {
        if (x3_wgrad_paired(g)) {
            in_ws = conv_wgrad_x3_workspace(&h);
        } else {   // SS wgrad over the 6 pairings, materialised from the parts
            in_ws = conv_tc_eligible(&h, DP_BF16, DP_CONV_WGRAD) ? conv_tc_workspace(&h, DP_CONV_WGRAD)
                                                                 : -1;
            wimg = 2 * align256(x3_operand_bytes(g, DP_X3_X)) +
                   2 * align256(x3_operand_bytes(g, DP_X3_XHALO)) +
                   2 * align256(x3_operand_bytes(g, DP_X3_DY));    // 6 blocks each
        }
    } else {
        wimg = align256(kParts * g->c_out * g->c_in * 9 * 2);
        in_ws = conv_tc_f32out_workspace(&h, which == DP_CONV_DGRAD);
    }
    if (wimg_bytes) *wimg_bytes = wimg;
    return in_ws < 0 ? -1 : wimg + align256(in_ws);
}

int launch_split(const float *x, int64_t B, int64_t C, int64_t S0, int64_t S1, const int64_t *st,
                 __nv_bfloat16 *out, int mode, int pat, cudaStream_t s) {
    if (B * C * S0 * S1 == 0) return DP_OK;
    const bool v4 = mode == 1 && pat == 1 && st[3] == 1 && S1 % 128 == 0 && C % 8 == 0 &&
                    st[0] % 4 == 0 && st[1] % 4 == 0 && st[2] % 4 == 0 &&
                    ((uintptr_t)x & 15) == 0;
    if (v4) {
        const int64_t nb = B * S0 * ((C + 31) / 32) * (S1 / 128);
        DP_REQUIRE(nb < (1ll << 31), DP_ERR_UNSUPPORTED, "x3 split: grid too large");
        x3_split_act_v4<<<(unsigned)nb, 256, 0, s>>>(x, B, C, S0, S1, st[0], st[1], st[2], out);
        return launch_status("x3_split_act_v4");
    }
    const int64_t blocks = B * S0 * ((C + 31) / 32) * ((S1 + 63) / 64);
    DP_REQUIRE(blocks < (1ll << 31), DP_ERR_UNSUPPORTED, "x3 split: grid too large");
    x3_split_act<<<(unsigned)blocks, 256, 0, s>>>(x, B, C, S0, S1, st[0], st[1], st[2], st[3], out,
                                                  mode, pat);
    return launch_status("x3_split_act");
}

// operand split: fp32 [B][C][S0][S1] (any strides) -> 3 bf16 parts as batch blocks
int x3_split_operand(const dp_conv_geom *g, int operand, const void *src, void *parts,
                     cudaStream_t st) {
    const int64_t *s = operand == DP_X3_X ? g->xs : operand == DP_X3_XHALO ? g->hs : g->ys;
    int64_t st4[4] = {s[0], s[1], s[2], s[3]};
    const int64_t C = operand == DP_X3_DY ? g->c_out : g->c_in;
    const int64_t S0 = operand == DP_X3_X ? g->in_ext[0]
                       : operand == DP_X3_XHALO ? g->halo : g->out_ext[0];
    const int64_t S1 = operand == DP_X3_DY ? g->out_ext[1] : g->in_ext[1];
    return launch_split((const float *)src, g->batch, C, S0, S1, st4, (__nv_bfloat16 *)parts, 1, 1,
                        st);
}

// fwd / dgrad / wgrad over split operands (a / ah / b as the `which` needs)
int x3_run(const dp_conv_geom *g, int which, const void *a, const void *ah, const void *b,
           void *out, void *out2, void *ws, int64_t ws_bytes, cudaStream_t st) {
    int64_t wimg = 0;
    const int64_t need = x3_inner_bytes(g, which, &wimg);
    DP_REQUIRE(need >= 0, DP_ERR_UNSUPPORTED, "conv_x3: outside the envelope");
    DP_REQUIRE(ws_bytes >= need, DP_ERR_INVALID, "conv_x3: workspace too small");
    uint8_t *w8 = (uint8_t *)ws;
    const dp_conv_geom h = x3_geom(g, which);
    int rc;
    if (which == DP_CONV_WGRAD && x3_wgrad_paired(g))  // a = x parts, ah = x halo parts, b = dy parts
        return conv_wgrad_x3_launch(&h, a, g->halo > 0 ? ah : nullptr, b, out, ws, ws_bytes, st,
                                    (int)g->batch);
    if (which == DP_CONV_WGRAD) {
        // the 6 pairings (X part c_ppat[k], dY part c_dpat[k]) as batch blocks
        static const int ppat[kParts] = {0, 1, 0, 2, 1, 0}, dpat[kParts] = {0, 0, 1, 0, 1, 2};
        const int64_t bx = x3_operand_bytes(g, DP_X3_X) / 3, bxh = x3_operand_bytes(g, DP_X3_XHALO) / 3,
                      bd = x3_operand_bytes(g, DP_X3_DY) / 3;
        uint8_t *x6 = w8, *xh6 = x6 + 2 * align256(3 * bx), *d6 = xh6 + 2 * align256(3 * bxh);
        for (int k = 0; k < kParts; ++k) {
            DP_CUDA_CHECK(cudaMemcpyAsync(x6 + k * bx, (const uint8_t *)a + ppat[k] * bx, bx,
                                          cudaMemcpyDeviceToDevice, st));
            if (g->halo > 0)
                DP_CUDA_CHECK(cudaMemcpyAsync(xh6 + k * bxh, (const uint8_t *)ah + ppat[k] * bxh, bxh,
                                              cudaMemcpyDeviceToDevice, st));
            DP_CUDA_CHECK(cudaMemcpyAsync(d6 + k * bd, (const uint8_t *)b + dpat[k] * bd, bd,
                                          cudaMemcpyDeviceToDevice, st));
        }
        return conv_wgrad_tc_launch(&h, x6, g->halo > 0 ? xh6 : nullptr, d6, out, w8 + wimg,
                                    ws_bytes - wimg, st);
    }
    __nv_bfloat16 *wi = (__nv_bfloat16 *)w8;
    const int64_t nw = g->c_out * g->c_in * 9;
    x3_split_weight<<<grid_for(nw, 256, 2), 256, 0, st>>>((const float *)b, g->c_out, g->c_in, 9,
                                                          wi, which == DP_CONV_DGRAD ? 1 : 0);
    if ((rc = launch_status("x3_split_weight"))) return rc;
    if (which == DP_CONV_FWD)     // a = x parts, ah = x halo parts, b = w (fp32), out = y
        return conv_tc_f32out_launch(&h, false, a, g->halo > 0 ? ah : nullptr, wi, out, nullptr,
                                     w8 + wimg, ws_bytes - wimg, st);
    // dgrad: a = dy parts, b = w (fp32), out = dx, out2 = dx halo
    return conv_tc_f32out_launch(&h, true, a, nullptr, wi, out, out2, w8 + wimg, ws_bytes - wimg,
                                 st);
}

// operand layout of the one-call path: the split operands, then the inner workspace
struct X3Layout {
    int64_t a, ah, b, inner, total;
};
X3Layout x3_layout(const dp_conv_geom *g, int which) {
    X3Layout L{};
    int64_t off = 0;
    if (which != DP_CONV_DGRAD) {
        L.a = off; off += align256(x3_operand_bytes(g, DP_X3_X));
        L.ah = off; off += align256(x3_operand_bytes(g, DP_X3_XHALO));
    }
    if (which != DP_CONV_FWD) {
        L.b = off; off += align256(x3_operand_bytes(g, DP_X3_DY));
    }
    L.inner = off;
    const int64_t in = x3_inner_bytes(g, which, nullptr);
    L.total = in < 0 ? -1 : off + in;
    return L;
}

}  // namespace

int conv_x3_eligible(const dp_conv_geom *g, int which) {
    if (!g || !x3_shape_ok(g)) return 0;
    return x3_inner_bytes(g, which, nullptr) >= 0 ? 1 : 0;
}

int64_t conv_x3_workspace(const dp_conv_geom *g, int which) {
    if (!conv_x3_eligible(g, which)) return -1;
    return x3_layout(g, which).total;
}

int64_t conv_x3_parts_workspace(const dp_conv_geom *g, int which) {
    if (!conv_x3_eligible(g, which)) return -1;
    return x3_inner_bytes(g, which, nullptr);
}

int64_t conv_x3_operand_bytes(const dp_conv_geom *g, int operand) {
    if (!g || !x3_shape_ok(g)) return -1;
    return x3_operand_bytes(g, operand);
}

int conv_x3_split(const dp_conv_geom *g, int operand, const void *src, void *parts,
                  cudaStream_t st) {
    DP_REQUIRE(g && x3_shape_ok(g), DP_ERR_UNSUPPORTED, "conv_x3_split: outside the envelope");
    DP_REQUIRE(operand == DP_X3_X || operand == DP_X3_XHALO || operand == DP_X3_DY, DP_ERR_INVALID,
               "conv_x3_split: unknown operand %d", operand);
    if (x3_operand_bytes(g, operand) == 0) return DP_OK;
    DP_REQUIRE(src && parts, DP_ERR_INVALID, "conv_x3_split: null buffer");
    return x3_split_operand(g, operand, src, parts, st);
}

int conv_x3_parts_launch(const dp_conv_geom *g, int which, const void *a, const void *ah,
                         const void *b, void *out, void *out2, void *ws, int64_t ws_bytes,
                         cudaStream_t st) {
    DP_REQUIRE(conv_x3_eligible(g, which), DP_ERR_UNSUPPORTED, "conv_x3: outside the envelope");
    return x3_run(g, which, a, ah, b, out, out2, ws, ws_bytes, st);
}

// one call: split the activation operands into the workspace, then run
int conv_x3_launch(const dp_conv_geom *g, int which, const void *a, const void *ah, const void *b,
                   void *out, void *out2, void *ws, int64_t ws_bytes, cudaStream_t st) {
    DP_REQUIRE(conv_x3_eligible(g, which), DP_ERR_UNSUPPORTED, "conv_x3: outside the envelope");
    const X3Layout L = x3_layout(g, which);
    DP_REQUIRE(L.total >= 0 && ws_bytes >= L.total, DP_ERR_INVALID, "conv_x3: workspace too small");
    uint8_t *w8 = (uint8_t *)ws;
    int rc;
    if (which == DP_CONV_DGRAD) {          // a = dy, b = w
        if ((rc = x3_split_operand(g, DP_X3_DY, a, w8 + L.b, st))) return rc;
        return x3_run(g, which, w8 + L.b, nullptr, b, out, out2, w8 + L.inner, ws_bytes - L.inner,
                      st);
    }
    if ((rc = x3_split_operand(g, DP_X3_X, a, w8 + L.a, st))) return rc;
    if (g->halo > 0 && (rc = x3_split_operand(g, DP_X3_XHALO, ah, w8 + L.ah, st))) return rc;
    if (which == DP_CONV_FWD)              // b = w
        return x3_run(g, which, w8 + L.a, w8 + L.ah, b, out, nullptr, w8 + L.inner,
                      ws_bytes - L.inner, st);
    if ((rc = x3_split_operand(g, DP_X3_DY, b, w8 + L.b, st))) return rc;   // wgrad: b = dy
    return x3_run(g, which, w8 + L.a, w8 + L.ah, w8 + L.b, out, nullptr, w8 + L.inner,
                  ws_bytes - L.inner, st);
}

}  // namespace dp
