"""Sharded hot path on one B200 with R thread-ranks: halo_conv fwd/bwd,
ring_attention fwd/bwd and redistribute against the reference's golden
outputs and the oracle."""

import json
import math

import numpy as np
import pytest
import torch

from conftest import load_npz, rel_err, to_np
from oracle import attention as oatt
from oracle import conv as oconv
from oracle import plan as oplan

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


def dp():
    import paper_2605_11111_b200 as m

    return m


def run(world, fn):
    return dp().spawn_mesh((world,), ("domain",), fn)


CONV = load_npz("conv_cases.npz")
RING = load_npz("ring_cases.npz")
REDIST = load_npz("redist_cases.npz")


@pytest.mark.parametrize("i", range(int(CONV["count"])))
def test_halo_conv_matches_reference_golden(i):
    """The reference's own halo_conv outputs (bitwise equal to its dense
    conv) vs ours: identical shard shapes, fp64 within 1e-12, fp32 1e-5."""
    m = dp()
    x, w, want = CONV[f"c{i}_x"], CONV[f"c{i}_w"], CONV[f"c{i}_y"]
    meta = json.loads(str(CONV[f"c{i}_meta"]))
    ext = tuple(meta["extents"])
    stride = meta["stride"] if isinstance(meta["stride"], int) else tuple(meta["stride"])
    pad = meta["padding"] if isinstance(meta["padding"], int) else tuple(meta["padding"])

    def prog(ctx):
        xt = torch.tensor(x) if ctx.rank_id == 0 else None
        st = m.scatter_global(ctx, xt, (m.Shard(meta["dim"]),), {0: ext})
        before = ctx.collective_count
        out = m.dispatch_operation("conv", st, torch.tensor(w, device=DEV), stride=stride,
                                   padding=pad)
        assert ctx.collective_count - before == 1
        assert ctx.trace[-1].line() == "op=conv level=aten_like collectives=1"
        return out.full_tensor(), out.shard_shapes[0]

    for full, shapes in run(len(ext), prog):
        assert list(shapes) == meta["out_extents"]
        tol = 1e-12 if x.dtype == np.float64 else 1e-5
        assert rel_err(to_np(full), want) < tol


CONV_SHARDED = [
    # global shape, kernel tail, stride, pad, shard dim, extents, dtype, channels_last
    ((1, 16, 16, 12, 20), (3, 3, 3), 1, 1, 2, (4, 4, 4, 4), torch.bfloat16, True),
    ((1, 16, 32, 8, 40), (3, 3, 3), 1, 1, 2, (5, 3, 9, 7, 8), torch.bfloat16, True),
    ((1, 32, 24, 6, 136), (3, 3, 3), 1, 1, 2, (3,) * 8, torch.bfloat16, True),
    ((1, 64, 40, 72), (3, 3), 1, 1, 2, (10, 10, 10, 10), torch.bfloat16, True),
    ((1, 32, 33, 47), (3, 3), 1, 1, 2, (17, 16), torch.float32, False),
    ((2, 3, 16, 18), (3, 3), 2, 1, 3, (5, 6, 7), torch.float32, False),
    # fp32 on the tensor cores with operands split once (bf16x3 parts in the tape):
    # c_out 16 (the SS wgrad over materialised pairings) with an empty shard, and
    # W = 256 (the float4 split path) over 3 uneven shards
    ((1, 16, 20, 130), (3, 3), 1, 1, 2, (8, 12, 0), torch.float32, False),
    ((1, 32, 12, 256), (3, 3), 1, 1, 2, (4, 5, 3), torch.float32, False),
    ((1, 4, 10, 12, 9), (3, 3, 3), 1, 1, 3, (4, 2, 6), torch.float64, False),
    ((1, 4, 10, 12, 9), (3, 3, 3), 1, 1, 4, (5, 4, 0), torch.float64, False),
]


@pytest.mark.parametrize("case", CONV_SHARDED)
def test_halo_conv_fwd_bwd_vs_oracle(case):
    """Sharded fwd against the fp64 oracle restatement, and the backward
    (dgrad + reverse halo + wgrad all-reduce) against the global gradient."""
    m = dp()
    shape, ktail, stride, pad, dim, ext, dtype, cl = case
    rng = np.random.default_rng(len(ext) * 100 + shape[1])
    x = rng.standard_normal(shape)
    w = rng.standard_normal((shape[1] if shape[1] <= 32 else 32, shape[1]) + ktail) * 0.1
    w = w[:32]
    xt = torch.tensor(x).to(dtype)
    wt = torch.tensor(w).to(dtype)
    xr, wr = to_np(xt).astype(np.float64), to_np(wt).astype(np.float64)
    want = oconv.conv(xr, wr, stride, pad)
    dy = rng.standard_normal(want.shape)
    dyt = torch.tensor(dy).to(dtype)
    dyr = to_np(dyt).astype(np.float64)
    dxr, dwr = oconv.conv_grads(xr, wr, dyr, stride, pad)
    plans = oplan.member_plans(list(ext), shape[dim], ktail[dim - 2],
                               stride if isinstance(stride, int) else stride[dim - 2],
                               pad if isinstance(pad, int) else pad[dim - 2])
    out_ext = [pl[1] - pl[0] for pl in plans]
    fmt = (torch.channels_last_3d if len(shape) == 5 else torch.channels_last) if cl else None

    def prog(ctx):
        st = m.scatter_global(ctx, xt if ctx.rank_id == 0 else None, (m.Shard(dim),), {0: ext})
        if fmt is not None:
            st = m.ShardTensor(st.local.contiguous(memory_format=fmt), st.global_shape, ctx,
                               st.placements, st.shard_shapes)
        out, tape = m.halo_conv_forward(st, wt.to(DEV), stride, pad)
        lo = sum(out_ext[:ctx.rank_id])
        dyl = dyt.narrow(dim, lo, out_ext[ctx.rank_id]).to(DEV)
        if fmt is not None:
            dyl = dyl.contiguous(memory_format=fmt)
        before = ctx.collective_count
        dx, dw = m.halo_conv_backward(tape, dyl)
        assert ctx.collective_count - before == 2
        return out.full_tensor(), dx.full_tensor(), dw, out.shard_shapes[0]

    tol = {torch.float64: 1e-12, torch.float32: 1e-5, torch.bfloat16: 1e-2}[dtype]
    for full, dx, dw, shapes in run(len(ext), prog):
        assert list(shapes) == out_ext
        assert rel_err(to_np(full), want) < tol
        assert rel_err(to_np(dx), dxr) < tol
        assert rel_err(to_np(dw), dwr) < (2e-2 if dtype == torch.bfloat16 else tol)


@pytest.mark.parametrize("i", range(int(RING["count"])))
def test_ring_attention_matches_reference_golden(i):
    m = dp()
    q, k, v, want = (RING[f"r{i}_{n}"] for n in ("q", "k", "v", "o"))
    qe, ke = tuple(int(a) for a in RING[f"r{i}_qe"]), tuple(int(a) for a in RING[f"r{i}_ke"])

    def prog(ctx):
        root = ctx.rank_id == 0
        qs = m.scatter_global(ctx, torch.tensor(q) if root else None, (m.Shard(0),), {0: qe})
        ks = m.scatter_global(ctx, torch.tensor(k) if root else None, (m.Shard(0),), {0: ke})
        vs = m.scatter_global(ctx, torch.tensor(v) if root else None, (m.Shard(0),), {0: ke})
        before = ctx.collective_count
        out = m.dispatch_operation("ring_attention", qs, ks, vs)
        assert ctx.collective_count - before == len(qe) - 1
        assert out.shard_shapes == qs.shard_shapes
        return out.full_tensor()

    tol = 1e-12 if q.dtype == np.float64 else 1e-5
    for full in run(len(qe), prog):
        assert np.isfinite(to_np(full)).all()
        assert rel_err(to_np(full), want) < tol


RING_BWD = [
    (12, 12, 1, 8, (5, 0, 4, 3), (5, 0, 4, 3), torch.float64),
    (19, 17, 2, 16, (3, 5, 4, 7), (9, 0, 0, 8), torch.float64),
    (64, 96, 2, 32, (16,) * 4, (24,) * 4, torch.float32),
    (256, 256, 4, 64, (32,) * 8, (32,) * 8, torch.bfloat16),
    (200, 300, 2, 64, (70, 0, 130), (100, 120, 80), torch.bfloat16),
]


@pytest.mark.parametrize("case", RING_BWD)
def test_ring_attention_fwd_bwd_vs_oracle(case):
    m = dp()
    sq, sk, h, d, qe, ke, dtype = case
    rng = np.random.default_rng(sq + sk)
    q = torch.tensor(rng.standard_normal((sq, h, d))).to(dtype)
    k = torch.tensor(rng.standard_normal((sk, h, d))).to(dtype)
    v = torch.tensor(rng.standard_normal((sk, h, d))).to(dtype)
    do = torch.tensor(rng.standard_normal((sq, h, d))).to(dtype)
    qr, kr, vr, dor = (to_np(t).astype(np.float64) for t in (q, k, v, do))
    want = oatt.sdpa(qr, kr, vr)
    dqr, dkr, dvr = oatt.sdpa_grads(qr, kr, vr, dor)
    qb = np.concatenate([[0], np.cumsum(qe)]).astype(int)

    def prog(ctx):
        root = ctx.rank_id == 0
        qs = m.scatter_global(ctx, q if root else None, (m.Shard(0),), {0: qe})
        ks = m.scatter_global(ctx, k if root else None, (m.Shard(0),), {0: ke})
        vs = m.scatter_global(ctx, v if root else None, (m.Shard(0),), {0: ke})
        out, tape = m.ring_attention_forward(qs, ks, vs)
        i = ctx.rank_id
        dq, dk, dv = m.ring_attention_backward(tape, do[qb[i]:qb[i + 1]].to(DEV))
        return out.full_tensor(), dq.full_tensor(), dk.full_tensor(), dv.full_tensor()

    tol = {torch.float64: 1e-11, torch.float32: 1e-5, torch.bfloat16: 2e-2}[dtype]
    for o, dq, dk, dv in run(len(qe), prog):
        assert rel_err(to_np(o), want) < tol
        assert rel_err(to_np(dq), dqr, 1.0) < tol
        assert rel_err(to_np(dk), dkr, 1.0) < tol
        assert rel_err(to_np(dv), dvr, 1.0) < tol


def _placements(m, names):
    out = []
    for n in names:
        out.append(m.Replicate() if n == "Replicate" else m.Shard(int(n[6:-1])))
    return tuple(out)


@pytest.mark.parametrize("i", range(int(REDIST["count"])))
def test_redistribute_bitexact_vs_reference(i):
    m = dp()
    meta = json.loads(str(REDIST[f"d{i}_meta"]))
    g = REDIST[f"d{i}_g"]
    mesh = tuple(meta["mesh"])
    names = ("domain",) if len(mesh) == 1 else ("a", "b")
    old, new = _placements(m, meta["old"]), _placements(m, meta["new"])
    shapes = None if meta["shapes"] is None else {int(a): tuple(v) for a, v in meta["shapes"].items()}

    def prog(ctx):
        st = m.scatter_global(ctx, torch.tensor(g) if ctx.rank_id == 0 else None, old, shapes)
        r = m.redistribute(st, new)
        return r.local, {a: list(v) for a, v in r.shard_shapes.items()}

    res = m.spawn_mesh(mesh, names, prog)
    for rank, (loc, sh) in enumerate(res):
        assert {str(a): v for a, v in sh.items()} == meta["out_shapes"]
        want = REDIST[f"d{i}_local{rank}"]
        assert tuple(loc.shape) == want.shape
        assert np.array_equal(to_np(loc), want)  # bit-exact


def test_two_d_mesh_data_x_domain():
    """(data, domain) = (2, 2) mesh: halo conv and ring attention use the
    domain-axis group only (domainpar/ops.py:328-338); dW is
    then averaged over the data axis (ddp_allreduce_grads, ops.py:429-444)."""
    m = dp()
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1, 16, 12, 6, 40))
    w = rng.standard_normal((32, 16, 3, 3, 3)) * 0.1
    q, k, v = (rng.standard_normal((300, 2, 64)) for _ in range(3))
    xt = torch.tensor(x).to(torch.bfloat16)
    wt = torch.tensor(w).to(torch.bfloat16)
    qt, kt, vt = (torch.tensor(a).to(torch.bfloat16) for a in (q, k, v))

    def prog(ctx):
        root = ctx.rank_id == 0
        pl = (m.Replicate(), m.Shard(2))
        st = m.scatter_global(ctx, xt if root else None, pl, {1: (7, 5)})
        st = m.ShardTensor(st.local.contiguous(memory_format=torch.channels_last_3d),
                           st.global_shape, ctx, st.placements, st.shard_shapes)
        before = ctx.collective_count
        y, tape = m.halo_conv_forward(st, wt.to(DEV), 1, 1)
        assert ctx.collective_count - before == 1
        o_ext = y.shard_shapes[1]
        lo = sum(o_ext[:ctx.coords[1]])
        dyl = torch.ones((1, 32, o_ext[ctx.coords[1]], 6, 40), dtype=torch.bfloat16,
                         device=DEV).contiguous(memory_format=torch.channels_last_3d)
        _, dw = m.halo_conv_backward(tape, dyl)
        dw_mean = m.ddp_allreduce_grads(ctx.axis_group("data"), [dw])[0]
        apl = (m.Replicate(), m.Shard(0))
        qs, ks, vs = (m.scatter_global(ctx, t if root else None, apl, {1: (120, 180)})
                      for t in (qt, kt, vt))
        o = m.ring_attention(qs, ks, vs)
        return y.full_tensor(), o.full_tensor(), dw, dw_mean, lo

    res = m.spawn_mesh((2, 2), ("data", "domain"), prog)
    xr, wr = to_np(xt).astype(np.float64), to_np(wt).astype(np.float64)
    want_y = oconv.conv(xr, wr, 1, 1)
    want_o = oatt.sdpa(*(to_np(t).astype(np.float64) for t in (qt, kt, vt)))
    for y, o, dw, dw_mean, _ in res:
        assert rel_err(to_np(y), want_y) < 1e-2
        assert rel_err(to_np(o), want_o) < 1.5e-2
        assert rel_err(to_np(dw_mean), to_np(dw)) < 1e-6   # data replicas agree
