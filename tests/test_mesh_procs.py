"""The one-process-per-rank transport (torch.distributed) with world size 2 on
CPU / gloo — the N > 1 path bench.py and init_mesh use with NCCL on GPUs.
Host tensors only (collectives, metadata, redistribute layouts); the device
kernels are covered by the GPU suite.  Mirrors the reference's mesh KATs
(pkg/tests/test_mesh.py:155-287, test_sharding.py:193-353)."""

import torch

import paper_2605_11111_b200 as dp
from paper_2605_11111_b200.errors import HaloError, MeshError


def run_procs(fn, world=2, **kw):
    return dp.spawn_mesh((world,), ("domain",), fn, backend="gloo", **kw)


def _varlen_prog(ctx):
    ext = (3, 0)
    lo = sum(ext[:ctx.rank_id])
    full = torch.arange(12.0).reshape(3, 4)
    local = full[lo:lo + ext[ctx.rank_id]].clone()
    g = ctx.axis_group()
    got = dp.all_gather_varlen(g, local, 0)
    return got, ctx.collective_count


def test_all_gather_varlen_uneven_and_empty_gloo():
    for got, count in run_procs(_varlen_prog):
        assert torch.equal(got, torch.arange(12.0).reshape(3, 4))
        assert count == 1


def _ring_prog(ctx):
    g = ctx.axis_group()
    x = torch.full((2, 3), float(ctx.rank_id))
    once = dp.ring_shift(g, x)
    twice = dp.ring_shift(g, once)
    return once, twice, ctx.collective_count


def test_ring_shift_cycles_gloo():
    res = run_procs(_ring_prog)
    for r, (once, twice, count) in enumerate(res):
        assert torch.equal(once, torch.full((2, 3), float((r - 1) % 2)))  # recv from index - 1
        assert torch.equal(twice, torch.full((2, 3), float(r)))
        assert count == 2


def _halo_prog(ctx):
    """pkg/tests/test_mesh.py:216-235: widths [(0,2),(1,0)] on a 10-column split."""
    full = torch.arange(30.0).reshape(3, 10)
    ext = (5, 5)
    lo = sum(ext[:ctx.rank_id])
    local = full[:, lo:lo + ext[ctx.rank_id]].clone()
    lw, rw = [(0, 2), (1, 0)][ctx.rank_id]
    return dp.halo_exchange(ctx.axis_group(), local, 1, lw, rw)


def test_halo_exchange_kat_gloo():
    full = torch.arange(30.0).reshape(3, 10)
    r0, r1 = run_procs(_halo_prog)
    assert torch.equal(r0, full[:, 0:7])
    assert torch.equal(r1, full[:, 4:10])


def _halo_too_wide(ctx):
    local = torch.zeros(2, 2 if ctx.rank_id == 1 else 5)
    lw, rw = [(0, 3), (0, 0)][ctx.rank_id]
    return dp.halo_exchange(ctx.axis_group(), local, 1, lw, rw)


def test_halo_single_hop_error_gloo():
    try:
        run_procs(_halo_too_wide, timeout=20)
    except MeshError as exc:
        err = exc.failures[1]
        assert isinstance(err, HaloError)
        assert "requested halo width 3" in str(err) and "single-hop" in str(err)
    else:
        raise AssertionError("expected MeshError")


def _redist_prog(ctx):
    """pkg/tests/test_sharding.py:278-311 on processes."""
    root = ctx.rank_id == 0
    st = dp.scatter_global(ctx, torch.arange(8.0).reshape(4, 2) if root else None,
                           (dp.Shard(0),), {0: (3, 1)})
    rep = dp.redistribute(st, (dp.Replicate(),))
    s1 = dp.redistribute(st, (dp.Shard(1),))
    full = dp.full_tensor(s1)
    return rep.local, s1.shard_shapes, s1.local, full, st.debug_line()


def test_redistribute_and_gather_gloo():
    res = run_procs(_redist_prog)
    g = torch.arange(8.0).reshape(4, 2)
    for r, (rep, shapes, s1, full, line) in enumerate(res):
        assert torch.equal(rep, g)
        assert shapes == {0: (1, 1)}
        assert torch.equal(s1, g[:, r:r + 1])
        assert torch.equal(full, g)
        assert line.startswith(f"rank={r}")


def _plan_prog(ctx):
    """halo_conv metadata on a process mesh: out extents and widths agree on
    every rank (replicated planning, no handshakes)."""
    pl = dp.halo_conv_plan([5, 5], 10, 3, 2, 1)
    return pl.out_extents, [(m.lw, m.rw) for m in pl.members]


def test_halo_plan_replicated_gloo():
    a, b = run_procs(_plan_prog)
    assert a == b
    assert a[0] == (3, 2)  # pkg/tests/test_acceptance.py:113-130


def _cl_halo_prog(ctx):
    """Channels-last blocks (the conv hot path's layout, batch 2 so a face is
    NOT one contiguous run): faces are packed in the block's own format,
    travel as bytes in memory order and land channels-last."""
    from paper_2605_11111_b200.mesh import halo_sendrecv

    ext = (5, 4)
    g = torch.arange(2 * 3 * 9 * 4 * 6, dtype=torch.float32).reshape(2, 3, 9, 4, 6)
    lo = sum(ext[:ctx.rank_id])
    local = g[:, :, lo:lo + ext[ctx.rank_id]].contiguous(memory_format=torch.channels_last_3d)
    grp = ctx.axis_group()
    serve_left = 2 if ctx.rank_id == 1 else 0
    rw = 2 if ctx.rank_id == 0 else 0
    lh, rh = halo_sendrecv(grp, local, 2, serve_left, 0, 0, rw)
    full = dp.full_tensor(dp.ShardTensor(local, tuple(g.shape), ctx, (dp.Shard(2),), {0: ext}))
    return (rh, None if rh is None else rh.is_contiguous(memory_format=torch.channels_last_3d),
            full, full.is_contiguous(memory_format=torch.channels_last_3d), g)


def test_channels_last_faces_over_gloo():
    res = run_procs(_cl_halo_prog)
    rh, is_cl, full, full_cl, g = res[0]
    assert is_cl and full_cl
    assert torch.equal(rh, g[:, :, 5:7])
    assert res[1][0] is None
    for _, _, full, _, g in res:
        assert torch.equal(full, g)
