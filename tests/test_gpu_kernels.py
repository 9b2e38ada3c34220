"""Device kernels vs the oracle: strided copy / accumulate, conv fwd/dgrad/
wgrad over the virtual halo block, attention block fold (SIMT and tcgen05)."""

import math

import numpy as np
import pytest
import torch

from conftest import rel_err, to_np
from oracle import attention as oatt
from oracle import conv as oconv

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


def kernels():
    from paper_2605_11111_b200 import kernels as k

    return k


LAYOUTS = [((1, 32, 6, 12, 40), torch.channels_last_3d, 2, 2),
           ((2, 16, 5, 9, 33), torch.channels_last_3d, 2, 3),
           ((3, 64, 7, 20), torch.channels_last, 2, 4),
           ((513, 16, 64), None, 0, 100)]


@pytest.mark.parametrize("shape,fmt,dim,n", LAYOUTS)
def test_element_maps_on_layouts(shape, fmt, dim, n):
    """copy / accumulate / convert / max / fill on channels-last and plain
    blocks and on their narrowed faces (the halo pack / unpack / reverse-halo
    shapes): exact against torch's own elementwise ops."""
    k = kernels()
    g = torch.Generator(device=DEV).manual_seed(3)

    def mk(dtype):
        t = torch.randn(shape, generator=g, device=DEV).to(dtype)
        return t.contiguous(memory_format=fmt) if fmt is not None else t

    for dtype in (torch.bfloat16, torch.float32, torch.float64):
        a, b = mk(dtype), mk(dtype)
        fa, fb = a.narrow(dim, 1, n), b.narrow(dim, 0, n)
        want = fa + fb if dtype != torch.bfloat16 else (fa.float() + fb.float()).to(dtype)
        k.accumulate(fa, fb)
        assert torch.equal(fa, want)
        want = torch.maximum(fa, fb)
        k.max_into(fa, fb)
        assert torch.equal(fa, want)
        dst = torch.empty_like(fb)
        k.copy_strided(dst, fb)
        assert torch.equal(dst, fb)
        for odt in (torch.bfloat16, torch.float32, torch.float64):
            o = torch.empty(fb.shape, dtype=odt, device=DEV)
            k.convert(o, fb)
            assert torch.equal(o, fb.to(odt))
        z = k.fill(torch.empty_like(a), -2.5)
        assert torch.equal(z, torch.full_like(a, -2.5))
        assert torch.equal(k.zeros(shape, dtype, DEV), torch.zeros(shape, dtype=dtype,
                                                                    device=DEV))


@pytest.mark.parametrize("shape,perm,sl", [
    ((64, 33, 7), (0, 1, 2), (slice(None), slice(3, 20), slice(None))),
    ((8, 16, 128), (2, 0, 1), (slice(None), slice(None), slice(5, 70))),
    ((1, 32, 9, 256, 256), (0, 1, 2, 3, 4), (slice(None), slice(None), slice(0, 2))),
    ((4, 4096), (0, 1), (slice(None), slice(1000, 3000))),
    ((3, 5, 7, 11), (3, 1, 0, 2), (slice(1, 3),)),
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64, torch.int64])
def test_copy_strided_matches_slicing(shape, perm, sl, dtype):
    src = torch.randn(shape, device=DEV).to(dtype) if dtype.is_floating_point else \
        torch.randint(-1000, 1000, shape, device=DEV, dtype=dtype)
    view = src.permute(perm)[sl] if len(sl) <= len(shape) else src.permute(perm)
    out = torch.empty(view.shape, dtype=dtype, device=DEV)
    kernels().copy_strided(out, view)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), view.cpu())  # bit-exact


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_accumulate_strided(dtype):
    base = torch.randn(4, 6, 10, device=DEV).to(dtype)
    add = torch.randn(4, 2, 10, device=DEV).to(dtype)
    want = base.clone().float()
    want[:, 1:3] += add.float()
    kernels().accumulate(base[:, 1:3], add)
    got = base.float()
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-6
    assert torch.allclose(got.cpu(), want.to(dtype).float().cpu(), atol=tol, rtol=tol)


def _conv_case(rng, nsp, batch, cin, cout, sp, k, s, p, dtype):
    x = rng.standard_normal((batch, cin) + sp)
    w = rng.standard_normal((cout, cin) + (k,) * nsp) * 0.3
    return x, w


CONV_CASES = [
    # nsp, batch, cin, cout, spatial, k, stride, pad
    (1, 2, 3, 4, (17,), 3, 1, 1),
    (1, 1, 2, 3, (20,), 5, 2, 3),
    (2, 2, 3, 5, (12, 9), 3, 1, 1),
    (2, 1, 4, 2, (11, 13), 5, 2, 2),
    (2, 1, 16, 32, (24, 40), 3, 1, 1),
    (3, 1, 4, 6, (7, 8, 9), 3, 1, 1),
    (3, 1, 16, 32, (6, 10, 20), 3, 1, 1),
    (3, 2, 3, 2, (7, 6, 9), 3, 2, 0),
]


def _layouts(x, channels_last):
    if not channels_last or x.dim() < 4:
        return x
    fmt = torch.channels_last if x.dim() == 4 else torch.channels_last_3d
    return x.contiguous(memory_format=fmt)


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("algo", ["simt", "auto"])
def test_dense_conv_fwd_bwd_vs_oracle(case, dtype, algo):
    """Unsharded conv: fwd, dgrad, wgrad against the fp64 oracle."""
    from paper_2605_11111_b200 import ops

    k = kernels()
    prev = k.set_algo(algo)
    try:
        nsp, batch, cin, cout, sp, ks, s, p = case
        rng = np.random.default_rng(hash(case) % 2**32)
        x, w = _conv_case(rng, nsp, batch, cin, cout, sp, ks, s, p, dtype)
        xt = _layouts(torch.tensor(x, device=DEV).to(dtype), algo == "auto")
        wt = torch.tensor(w, device=DEV).to(dtype)
        y = ops.dense_conv(xt, wt, s, p)
        # oracle on the (rounded) inputs, fp64
        xr, wr = to_np(xt).astype(np.float64), to_np(wt).astype(np.float64)
        want = oconv.conv(xr, wr, s, p)
        tol = {torch.float64: 1e-12, torch.float32: 1e-5, torch.bfloat16: 1e-2}[dtype]
        assert rel_err(to_np(y), want) < tol
        dy = rng.standard_normal(want.shape)
        dyt = _layouts(torch.tensor(dy, device=DEV).to(dtype), algo == "auto")
        from paper_2605_11111_b200.sharding import ShardTensor
        from paper_2605_11111_b200 import spawn_mesh, replicated

        def prog(ctx):
            xs = replicated(ctx, xt)
            out, tape = ops.halo_conv_forward(xs, wt, s, p)
            dx, dw = ops.halo_conv_backward(tape, dyt)
            return dx.local, dw

        dx, dw = spawn_mesh((1,), ("domain",), prog)[0]
        dxr, dwr = oconv.conv_grads(xr, wr, to_np(dyt).astype(np.float64), s, p)
        assert rel_err(to_np(dx), dxr) < tol
        assert rel_err(to_np(dw), dwr) < (tol if dtype != torch.bfloat16 else 2e-2)
    finally:
        k.set_algo(prev)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("sq,sk,h,d", [(5, 11, 1, 6), (37, 50, 3, 16), (130, 260, 2, 64),
                                        (64, 128, 4, 128), (1, 1, 1, 4)])
def test_attention_block_fold_vs_oracle(dtype, sq, sk, h, d):
    """Fold K/V in 3 uneven blocks through the state kernel == dense sdpa."""
    from paper_2605_11111_b200 import ops

    rng = np.random.default_rng(sq * 7 + sk)
    q = torch.tensor(rng.standard_normal((sq, h, d)), device=DEV).to(dtype)
    k_ = torch.tensor(rng.standard_normal((sk, h, d)), device=DEV).to(dtype)
    v = torch.tensor(rng.standard_normal((sk, h, d)), device=DEV).to(dtype)
    cuts = [0, sk // 3, sk // 3, sk]  # includes an empty block
    blocks = [(k_[a:b], v[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    out, lse = ops._attn_local(q, blocks, 1.0 / math.sqrt(d))
    want = oatt.sdpa(to_np(q).astype(np.float64), to_np(k_).astype(np.float64),
                     to_np(v).astype(np.float64))
    tol = {torch.float64: 1e-12, torch.float32: 1e-5, torch.bfloat16: 1.5e-2}[dtype]
    assert rel_err(to_np(out), want) < tol


TC_CASES = [
    # nsp, batch, cin, cout, spatial, k, pad, halo_rows (sharded virtual block)
    (3, 1, 16, 32, (5, 7, 200), 3, 1, 0),
    (3, 1, 32, 32, (4, 9, 130), 3, 1, 2),
    (3, 2, 16, 16, (3, 5, 64), 3, 1, 1),
    (2, 1, 64, 64, (40, 300), 3, 1, 2),
    (2, 1, 32, 48, (9, 129), 3, 1, 0),
    (2, 1, 16, 32, (12, 70), 5, 2, 4),
    (3, 1, 16, 48, (3, 4, 128), 3, 1, 0),
    # C_out = 32, 3x3(x3): the TS-form wgrad (dY in TMEM) with 1, 2 and 3 w' tiles
    (3, 2, 32, 32, (3, 6, 256), 3, 1, 1),
    (2, 1, 32, 32, (10, 260), 3, 1, 1),
    (2, 1, 64, 32, (7, 100), 3, 1, 0),
    (2, 1, 16, 32, (5, 33), 3, 0, 0),
    (3, 1, 16, 32, (4, 3, 300), 3, 1, 2),
    # rows of 161..256 voxels with padding 1: the CTA-pair (cta_group::2) fwd/dgrad
    (3, 1, 16, 32, (4, 5, 256), 3, 1, 2),
    (3, 1, 32, 16, (3, 4, 200), 3, 1, 1),
    (2, 1, 32, 32, (6, 256), 3, 1, 0),
    (3, 2, 16, 16, (3, 3, 181), 3, 1, 1),
    (2, 2, 16, 32, (5, 170), 3, 1, 3),
    # 64 -> 64 2-D rows of 200..256 voxels: the N = 64 CTA-pair fwd / dgrad (cfg4's layers)
    (2, 1, 64, 64, (6, 256), 3, 1, 2),
    (2, 2, 64, 64, (5, 200), 3, 1, 0),
    # 3-D odd output-plane counts with a halo: the P-pair units' last, half-empty pair
    (3, 1, 16, 32, (5, 4, 256), 3, 1, 2),
    (3, 1, 32, 16, (3, 6, 140), 3, 1, 1),
]


@pytest.mark.parametrize("case", TC_CASES)
def test_conv_tc_fwd_dgrad_vs_oracle(case):
    """tcgen05 path forced (DP_ALGO_TC): forward and dgrad over the virtual
    block [main | halo | zeros] on the sharded (outermost spatial) dim."""
    k = kernels()
    nsp, batch, cin, cout, sp, ks, pad, hrows = case
    rng = np.random.default_rng(sum(sp) + cin)
    fmt = torch.channels_last_3d if nsp == 3 else torch.channels_last
    full_sp = (sp[0] + hrows,) + sp[1:]
    xfull = torch.tensor(rng.standard_normal((batch, cin) + full_sp)).to(torch.bfloat16)
    w = torch.tensor(rng.standard_normal((cout, cin) + (ks,) * nsp) * 0.1).to(torch.bfloat16)
    x = xfull[:, :, :sp[0]].to(DEV).contiguous(memory_format=fmt)
    xh = xfull[:, :, sp[0]:].to(DEV).contiguous(memory_format=fmt) if hrows else None
    # a rank at the global start: outputs cover [0, sp0 + hrows - ks + 1 + pad) on dim 0
    g_lo = -pad
    n0 = sp[0] + hrows - ks + 1 + pad
    out_sp = (n0,) + tuple(e + 2 * pad - ks + 1 for e in sp[1:])
    y = torch.empty((batch, cout) + out_sp, dtype=torch.bfloat16, device=DEV,
                    memory_format=fmt)
    prev = k.set_algo("tc")
    try:
        base = [g_lo] + [-pad] * (nsp - 1)
        k.conv_fwd(x, xh, w.to(DEV).contiguous(), y, kernel=(ks,) * nsp, stride=(1,) * nsp,
                   base=base, shard=0, halo_rows=hrows)
        # oracle: global conv over [main | halo] padded, rows [0, n0)
        xr = to_np(xfull).astype(np.float64)
        wr = to_np(w).astype(np.float64)
        big = np.pad(xr, [(0, 0), (0, 0), (pad, 0)] + [(pad, pad)] * (nsp - 1))
        want = oconv.conv(big, wr, 1, (0,) + (0,) * (nsp - 1))[:, :, :n0]
        assert rel_err(to_np(y), want) < 1e-2
        # dgrad of this virtual conv
        dy = torch.tensor(rng.standard_normal(tuple(y.shape))).to(torch.bfloat16)
        dyd = dy.to(DEV).contiguous(memory_format=fmt)
        dx = torch.empty(x.shape, dtype=torch.bfloat16, device=DEV, memory_format=fmt)
        dxh = torch.empty(xh.shape, dtype=torch.bfloat16, device=DEV,
                          memory_format=fmt) if hrows else None
        k.conv_dgrad(dyd, w.to(DEV).contiguous(), dx, dxh, kernel=(ks,) * nsp,
                     stride=(1,) * nsp, base=base, shard=0, halo_rows=hrows)
        gx, _ = oconv.conv_grads(big[:, :, :n0 + ks - 1], wr, to_np(dy).astype(np.float64), 1, 0)
        gx = gx[:, :, pad:]  # drop the virtual zero rows at the global start
        gx = gx[(slice(None), slice(None), slice(None)) + tuple(slice(pad, pad + e) for e in sp[1:])]
        got = to_np(dx)
        if hrows:
            got = np.concatenate([got, to_np(dxh)], axis=2)
        assert rel_err(got, gx[:, :, :got.shape[2]]) < 1e-2
        # wgrad of the same virtual conv (fp32 partial, no all-reduce here)
        dw = torch.empty(w.shape, dtype=torch.float32, device=DEV)
        k.conv_wgrad(x, xh, dyd, dw, kernel=(ks,) * nsp, stride=(1,) * nsp, base=base, shard=0,
                     halo_rows=hrows)
        _, gw = oconv.conv_grads(big[:, :, :n0 + ks - 1], wr, to_np(dy).astype(np.float64), 1, 0)
        assert rel_err(to_np(dw), gw) < 1e-3
    finally:
        k.set_algo(prev)


ATTN_TC_CASES = [
    # sq, sk, heads, key-block cuts (ring steps folded one after another)
    (128, 128, 1, [128]),
    (200, 300, 2, [0, 37, 300]),          # partial tiles, an uneven split
    (1000, 513, 3, [100, 100, 513]),      # includes an empty block (no-op)
    (64, 1030, 2, [1030]),
    (384, 256, 4, [1, 256]),              # a one-key block
    (700, 640, 2, [640]),                 # 6 query blocks: Q/dO ring + LSE/D ring wrap
    (2048, 384, 1, [200, 384]),           # 16 query blocks, ragged key tiles
]


@pytest.mark.parametrize("case", ATTN_TC_CASES)
@pytest.mark.parametrize("payload", [False, True])
def test_attention_tc_fwd_bwd_vs_oracle(case, payload):
    """tcgen05 path forced: forward fold + finalize and the backward block
    over K/V blocks taken from the ring's [S, 2, H, d] K||V payload (strided
    views) or from plain tensors; bf16, d = 64; vs fp64 oracle."""
    k = kernels()
    sq, sk, h, cuts = case
    d = 64
    rng = np.random.default_rng(sq * 7 + sk)
    q, kk, v, do = (torch.tensor(rng.standard_normal((n, h, d))).to(torch.bfloat16)
                    for n in (sq, sk, sk, sq))
    qd = q.to(DEV)
    if payload:
        pay = torch.stack([kk, v], dim=1).to(DEV)  # [sk, 2, H, d]
        kd, vd = pay[:, 0], pay[:, 1]
    else:
        kd, vd = kk.to(DEV), v.to(DEV)
    dod = do.to(DEV)
    scale = 1.0 / math.sqrt(d)
    bounds = [0] + [c for c in cuts]
    bounds = sorted(set(min(b, sk) for b in bounds) | {sk})
    prev = k.set_algo("tc")
    try:
        m = torch.full((sq, h), -math.inf, device=DEV)
        l = torch.zeros((sq, h), device=DEV)
        acc = torch.zeros((sq, h, d), device=DEV)
        for a, b in zip(bounds[:-1], bounds[1:]):
            k.attn_fwd_update(qd, kd[a:b], vd[a:b], m, l, acc, scale)
        out = torch.empty_like(qd)
        lse = torch.empty_like(m)
        k.attn_finalize(qd, m, l, acc, out, lse, 1.0)
        delta = torch.empty((sq, h), device=DEV)
        k.attn_bwd_preprocess(out, dod, delta)
        dq = torch.zeros((sq, h, d), device=DEV)
        dk = torch.zeros((sk, h, d), device=DEV)
        dv = torch.zeros_like(dk)
        for a, b in zip(bounds[:-1], bounds[1:]):
            k.attn_bwd_update(qd, kd[a:b], vd[a:b], dod, lse, delta, dq, dk[a:b], dv[a:b], scale)
        torch.cuda.synchronize()
    finally:
        k.set_algo(prev)
    qr, kr, vr, dr = (to_np(t).astype(np.float64) for t in (q, kk, v, do))
    assert rel_err(to_np(out), oatt.sdpa(qr, kr, vr)) < 1.5e-2
    for got, want in zip((dq, dk, dv), oatt.sdpa_grads(qr, kr, vr, dr)):
        assert rel_err(to_np(got), want, floor=1.0) < 1.5e-2


def test_conv_single_cta_and_per_mma_issue_paths():
    """The non-default conv issue paths stay correct: single-CTA MMAs
    (DP_CONV_2CTA=0) and one elect per MMA instead of the grouped kw taps
    (DP_CONV_DBG=32), each over the tcgen05 conv parity cases."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    for env_extra in ({"DP_CONV_2CTA": "0"}, {"DP_CONV_DBG": "32"}):
        env = dict(os.environ, **env_extra)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x",
                            os.path.join(here, "test_gpu_kernels.py"),
                            "-k", "test_conv_tc_fwd_dgrad_vs_oracle"], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, str(env_extra) + r.stdout[-2000:] + r.stderr[-2000:]


X3_CASES = [
    # batch, cin, cout, (H, W), pad, halo rows: fp32 convs on the bf16x3 tensor-core path
    (1, 32, 32, (40, 300), 1, 0),
    (2, 16, 32, (21, 77), 1, 2),
    (1, 32, 16, (9, 130), 0, 2),
    (1, 16, 16, (12, 33), 1, 1),
]


@pytest.mark.parametrize("case", X3_CASES)
def test_conv_fp32_bf16x3_vs_oracle(case):
    """fp32 fwd / dgrad / wgrad on the tensor cores through three-way bf16
    splits (conv_x3.cu) hold the reference's fp32 tolerance (1e-5) against the
    fp64 oracle, over the virtual [main | halo] block."""
    k = kernels()
    batch, cin, cout, sp, pad, hrows = case
    rng = np.random.default_rng(cin * 7 + sp[1])
    full = (sp[0] + hrows, sp[1])
    xfull = torch.tensor(rng.standard_normal((batch, cin) + full)).float()
    w = torch.tensor(rng.standard_normal((cout, cin, 3, 3)) * 0.1).float()
    x = xfull[:, :, :sp[0]].to(DEV).contiguous()
    xh = xfull[:, :, sp[0]:].to(DEV).contiguous() if hrows else None
    n0 = sp[0] + hrows - 3 + 1 + pad
    out_sp = (n0, sp[1] + 2 * pad - 2)
    y = torch.empty((batch, cout) + out_sp, device=DEV)
    base = [-pad, -pad]
    prev = k.set_algo("tc")
    try:
        k.conv_fwd(x, xh, w.to(DEV), y, kernel=(3, 3), stride=(1, 1), base=base, shard=0,
                   halo_rows=hrows)
        xr, wr = to_np(xfull).astype(np.float64), to_np(w).astype(np.float64)
        big = np.pad(xr, [(0, 0), (0, 0), (pad, 0), (pad, pad)])
        want = oconv.conv(big, wr, 1, 0)[:, :, :n0]
        assert rel_err(to_np(y), want) < 1e-5
        dy = torch.tensor(rng.standard_normal(tuple(y.shape))).float()
        dx = torch.empty(x.shape, device=DEV)
        dxh = torch.empty(xh.shape, device=DEV) if hrows else None
        k.conv_dgrad(dy.to(DEV), w.to(DEV), dx, dxh, kernel=(3, 3), stride=(1, 1), base=base,
                     shard=0, halo_rows=hrows)
        gx, gw = oconv.conv_grads(big[:, :, :n0 + 2], wr, to_np(dy).astype(np.float64), 1, 0)
        gx = gx[:, :, pad:, pad:pad + sp[1]]
        got = to_np(dx) if not hrows else np.concatenate([to_np(dx), to_np(dxh)], axis=2)
        assert rel_err(got, gx[:, :, :got.shape[2]]) < 1e-5
        dw = torch.empty(w.shape, device=DEV)
        k.conv_wgrad(x, xh, dy.to(DEV), dw, kernel=(3, 3), stride=(1, 1), base=base, shard=0,
                     halo_rows=hrows)
        assert rel_err(to_np(dw), gw) < 1e-5
    finally:
        k.set_algo(prev)


@pytest.mark.parametrize("shape,op", [((2, 32, 5, 256), 0), ((1, 16, 3, 384), 2),
                                      ((2, 32, 4, 200), 0), ((1, 32, 2, 128), 1)])
def test_x3_split_parts_bitexact(shape, op):
    """dp_conv_x3_split: the 3 bf16 parts of every fp32 value, exactly
    (x = xh + xm + xl, each the bf16 rounding of the remainder), laid out as
    batch blocks [3][B][s0][s1][C] — float4 tile path (W % 128 == 0) and the
    scalar tile path (W = 200)."""
    k = kernels()
    B, C, S0, S1 = shape
    g = torch.Generator().manual_seed(sum(shape))
    x = (torch.randn(shape, generator=g) * torch.logspace(-3, 3, S1)).to(DEV)
    c_out = 32
    if op == k.X3_DY:      # dy of a conv with C output channels: geometry over x of c_in = 32
        xg = torch.empty((B, 32, S0, S1), device=DEV)
        w_out = C
        geom = k.conv_geom(xg, None, x.shape, x.stride(), w_out, (3, 3), (1, 1), (-1, -1), 0, 0)
    elif op == k.X3_XHALO:
        xg = torch.empty((B, C, 7, S1), device=DEV)
        geom = k.conv_geom(xg, x, (B, c_out, 7, S1), (7 * S1 * c_out, 1, S1 * c_out, c_out),
                           c_out, (3, 3), (1, 1), (0, -1), 0, S0)
    else:
        geom = k.conv_geom(x, None, (B, c_out, S0, S1), (S0 * S1 * c_out, 1, S1 * c_out, c_out),
                           c_out, (3, 3), (1, 1), (-1, -1), 0, 0)
    parts = k.x3_split(x, op, geom).view(3, B, S0, S1, C)
    xh = x.to(torch.bfloat16)
    r1 = x - xh.float()
    xm = r1.to(torch.bfloat16)
    xl = (r1 - xm.float()).to(torch.bfloat16)
    want = torch.stack([t.permute(0, 2, 3, 1) for t in (xh, xm, xl)])
    assert torch.equal(parts.view(torch.int16), want.contiguous().view(torch.int16))
