"""Mesh, collectives and ShardTensor metadata on the thread mesh with host
tensors (the reference's own test model, pkg/tests/test_mesh.py and
test_sharding.py) — host-side logic only; no device arithmetic."""

import json

import numpy as np
import pytest
import torch

import paper_2605_11111_b200 as dp
from paper_2605_11111_b200.errors import (CollectiveError, DimensionError, HaloError,
                                          IntegrityError, MeshError, MetadataError)

CPU = torch.device("cpu")


def run1d(world, fn, **kw):
    return dp.spawn_mesh((world,), ("domain",), fn, device=CPU, **kw)


def test_mesh_geometry():
    m = dp.DeviceMesh((2, 3), ("a", "b"))
    assert m.world_size == 6
    assert [m.coords_of(r) for r in range(6)] == [(0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (1, 2)]
    assert all(m.rank_of(m.coords_of(r)) == r for r in range(6))
    with pytest.raises(DimensionError):
        dp.DeviceMesh((2, 2, 2), ("a", "b", "c"))
    with pytest.raises(DimensionError):
        dp.DeviceMesh((2,), ("a", "b"))


def test_axis_groups_2d():
    def prog(ctx):
        ga, gb = ctx.axis_group("a"), ctx.axis_group("b")
        return ga.members, ga.index, gb.members, gb.index

    res = dp.spawn_mesh((2, 3), ("a", "b"), prog, device=CPU)
    assert res[4] == ((1, 4), 1, (3, 4, 5), 1)


def test_all_reduce_sum_max_bitwise_identical():
    def prog(ctx):
        g = ctx.axis_group()
        x = torch.tensor([0.1 * (ctx.rank_id + 1), -ctx.rank_id], dtype=torch.float64)
        return dp.all_reduce(g, x, "sum"), dp.all_reduce(g, x, "max"), ctx.collective_count

    res = run1d(4, prog)
    for s, mx, c in res:
        assert torch.equal(s, res[0][0]) and c == 2
        assert mx.tolist() == [0.4, 0.0]
    with pytest.raises(MeshError, match="all_reduce op"):
        run1d(2, lambda ctx: dp.all_reduce(ctx.axis_group(), torch.zeros(1), "min"))


def test_all_gather_varlen_uneven_and_empty():
    ext = (3, 0, 2, 1)

    def prog(ctx):
        lo = sum(ext[:ctx.rank_id])
        local = torch.arange(lo, lo + ext[ctx.rank_id], dtype=torch.float32).reshape(-1, 1)
        return dp.all_gather_varlen(ctx.axis_group(), local.expand(-1, 2).contiguous(), 0)

    for out in run1d(4, prog):
        assert out[:, 0].tolist() == [0, 1, 2, 3, 4, 5]


def test_all_gather_varlen_mismatch_raises():
    def prog(ctx):
        return dp.all_gather_varlen(ctx.axis_group(), torch.zeros(2, 1 + ctx.rank_id), 0)

    with pytest.raises(MeshError, match="mismatch"):
        run1d(2, prog)


def test_ring_shift_cycles():
    for world in (1, 2, 5):
        def prog(ctx):
            return dp.ring_shift(ctx.axis_group(), torch.full((ctx.rank_id + 1,), ctx.rank_id))

        res = run1d(world, prog)
        for r, got in enumerate(res):
            src = (r - 1) % world
            assert got.tolist() == [src] * (src + 1)


# halo KATs: pkg/tests/test_mesh.py:216-287
def test_halo_exchange_asymmetric_widths():
    full = torch.arange(20, dtype=torch.float64).reshape(2, 10)
    widths = [(0, 2), (1, 0)]

    def prog(ctx):
        lo = 5 * ctx.rank_id
        lw, rw = widths[ctx.rank_id]
        out = dp.halo_exchange(ctx.axis_group(), full[:, lo:lo + 5].clone(), 1, lw, rw)
        assert ctx.collective_count == 1
        return out

    r0, r1 = run1d(2, prog)
    assert torch.equal(r0, full[:, 0:7]) and torch.equal(r1, full[:, 4:10])


def test_halo_exchange_interior_rank_both_sides():
    full = torch.arange(12, dtype=torch.float64)
    widths = [(0, 1), (2, 1), (1, 0)]

    def prog(ctx):
        lo = 4 * ctx.rank_id
        lw, rw = widths[ctx.rank_id]
        return dp.halo_exchange(ctx.axis_group(), full[lo:lo + 4].clone(), 0, lw, rw)

    r0, r1, r2 = run1d(3, prog)
    assert torch.equal(r0, full[0:5]) and torch.equal(r1, full[2:9]) and torch.equal(r2, full[7:12])


def test_halo_exchange_zero_widths_and_single_rank():
    res = run1d(3, lambda ctx: dp.halo_exchange(ctx.axis_group(), torch.full((3,), 1.0), 0, 0, 0))
    assert all(r.tolist() == [1.0] * 3 for r in res)
    res = run1d(1, lambda ctx: dp.halo_exchange(ctx.axis_group(), torch.arange(4.0), 0, 0, 0))
    assert res[0].tolist() == [0, 1, 2, 3]


def test_halo_wider_than_neighbor_is_an_error():
    ext = (5, 2)
    widths = [(0, 3), (0, 0)]

    def prog(ctx):
        lw, rw = widths[ctx.rank_id]
        return dp.halo_exchange(ctx.axis_group(), torch.zeros(ext[ctx.rank_id]), 0, lw, rw)

    with pytest.raises(MeshError) as info:
        run1d(2, prog)
    msg = str(info.value)
    assert "rank 0 requested halo width 3 from rank 1" in msg
    assert "holds only 2" in msg and "single-hop" in msg
    assert isinstance(info.value.failures[1], HaloError)


def test_halo_negative_width_rejected():
    with pytest.raises(MeshError, match="widths must be >= 0"):
        run1d(2, lambda ctx: dp.halo_exchange(ctx.axis_group(), torch.zeros(3), 0, -1, 0))


def test_failure_unwinds_and_names_primary():
    def prog(ctx):
        if ctx.rank_id == 1:
            raise ValueError("boom")
        return dp.all_gather_varlen(ctx.axis_group(), torch.zeros(1), 0)

    with pytest.raises(MeshError) as info:
        run1d(3, prog, timeout=10)
    assert "1 rank(s) failed" in str(info.value) and "boom" in str(info.value)


def test_receive_timeout():
    def prog(ctx):
        if ctx.rank_id == 0:
            return dp.ring_shift(ctx.axis_group(), torch.zeros(1))
        import time

        time.sleep(1.0)
        return None

    with pytest.raises(MeshError, match="timed out|finished without"):
        run1d(2, prog, timeout=0.3)


def test_timeout_env(monkeypatch):
    monkeypatch.setenv("DP_COLLECTIVE_TIMEOUT_SECS", "nope")
    with pytest.raises(DimensionError):
        run1d(1, lambda ctx: 0)


# ShardTensor metadata: pkg/tests/test_sharding.py


def test_debug_lines_match_reference(plans_golden):
    def prog(ctx):
        root = ctx.rank_id == 0
        st = dp.scatter_global(ctx, torch.zeros(5, 3) if root else None, (dp.Shard(0),),
                               {0: (3, 0, 2)})
        rep = dp.replicated(ctx, torch.arange(4.0))
        return st.debug_line(), rep.debug_line()

    assert [list(x) for x in run1d(3, prog)] == plans_golden["debug_lines"]

    def prog2(ctx):
        root = ctx.rank_id == 0
        st = dp.scatter_global(ctx, torch.zeros(4, 6) if root else None,
                               (dp.Shard(0), dp.Shard(1)))
        return st.debug_line()

    assert dp.spawn_mesh((2, 3), ("a", "b"), prog2, device=CPU) == plans_golden["debug_lines_2d"]


def test_metadata_errors():
    def prog(ctx):
        with pytest.raises(MetadataError, match="placements"):
            dp.ShardTensor(torch.zeros(2), (4,), ctx, (dp.Shard(0), dp.Replicate()))
        with pytest.raises(MetadataError, match="sum to"):
            dp.ShardTensor(torch.zeros(2), (4,), ctx, (dp.Shard(0),), {0: (2, 1)})
        with pytest.raises(IntegrityError, match="local shape"):
            dp.ShardTensor(torch.zeros(3), (4,), ctx, (dp.Shard(0),), {0: (2, 2)})
        with pytest.raises(MetadataError, match="do not match"):
            dp.ShardTensor(torch.zeros(2), (4,), ctx, (dp.Shard(0),), {})
        return True

    assert all(run1d(2, prog))

    def prog2(ctx):
        with pytest.raises(MetadataError, match="more than one"):
            dp.ShardTensor(torch.zeros(2, 2), (2, 4), ctx, (dp.Shard(1), dp.Shard(1)))
        return True

    assert all(dp.spawn_mesh((2, 2), ("a", "b"), prog2, device=CPU))


def test_scatter_full_round_trip_uneven():
    g = torch.arange(24.0).reshape(6, 4)

    def prog(ctx):
        st = dp.scatter_global(ctx, g if ctx.rank_id == 0 else None, (dp.Shard(0),),
                               {0: (3, 0, 2, 1)})
        before = ctx.collective_count
        full = dp.full_tensor(st)
        assert ctx.collective_count - before == 1
        return st.shard_interval(0), full

    for r, (iv, full) in enumerate(run1d(4, prog)):
        assert torch.equal(full, g)
    assert run1d(4, prog)[2][0] == (3, 5)


def test_scatter_bad_shapes_rejected_on_root():
    def prog(ctx):
        return dp.scatter_global(ctx, torch.zeros(5) if ctx.rank_id == 0 else None,
                                 (dp.Shard(0),), {0: (2, 2)})

    with pytest.raises(MeshError, match="do not tile"):
        run1d(2, prog, timeout=2)


def test_full_tensor_2d_mesh():
    g = torch.arange(48.0).reshape(6, 8)

    def prog(ctx):
        st = dp.scatter_global(ctx, g if ctx.rank_id == 0 else None, (dp.Shard(0), dp.Shard(1)),
                               {0: (5, 1), 1: (3, 0, 5)})
        return dp.full_tensor(st)

    for full in dp.spawn_mesh((2, 3), ("a", "b"), prog, device=CPU):
        assert torch.equal(full, g)


def test_redistribute_host_kats():
    """pkg/tests/test_sharding.py:278-353."""
    def prog(ctx):
        root = ctx.rank_id == 0
        st = dp.scatter_global(ctx, torch.arange(8.0).reshape(4, 2) if root else None,
                               (dp.Shard(0),), {0: (3, 1)})
        assert dp.redistribute(st, (dp.Shard(0),)) is st
        before = ctx.collective_count
        rep = dp.redistribute(st, (dp.Replicate(),))
        assert ctx.collective_count - before == 1
        back = dp.redistribute(rep, (dp.Shard(1),))
        assert ctx.collective_count - before == 1  # Replicate -> Shard is local
        s1 = dp.redistribute(st, (dp.Shard(1),))
        return rep.local, back.shard_shapes, s1.shard_shapes, s1.local

    res = run1d(2, prog)
    for r, (rep, bs, s1s, s1) in enumerate(res):
        assert torch.equal(rep, torch.arange(8.0).reshape(4, 2))
        assert bs == {0: (1, 1)} and s1s == {0: (1, 1)}
        assert torch.equal(s1, torch.arange(8.0).reshape(4, 2)[:, r:r + 1])


def test_redistribute_contiguous_host_path_vs_golden():
    """Cases whose packs are contiguous on the host (gather to Replicate)."""
    from conftest import load_npz

    d = load_npz("redist_cases.npz")
    checked = 0
    for i in range(int(d["count"])):
        meta = json.loads(str(d[f"d{i}_meta"]))
        if meta["mesh"] != [meta["mesh"][0]] or meta["new"] != ["Replicate"]:
            continue
        g = torch.tensor(d[f"d{i}_g"])
        shapes = {int(a): tuple(v) for a, v in meta["shapes"].items()}
        old = (dp.Shard(int(meta["old"][0][6:-1])),)

        def prog(ctx, g=g, shapes=shapes, old=old):
            st = dp.scatter_global(ctx, g if ctx.rank_id == 0 else None, old, shapes)
            return dp.redistribute(st, (dp.Replicate(),)).local

        for rank, loc in enumerate(run1d(meta["mesh"][0], prog)):
            assert np.array_equal(loc.numpy(), d[f"d{i}_local{rank}"])
        checked += 1
    assert checked >= 3


def test_collective_error_on_finished_peer():
    def prog(ctx):
        if ctx.rank_id == 1:
            return None
        return dp.all_gather_varlen(ctx.axis_group(), torch.zeros(1), 0)

    with pytest.raises(MeshError) as info:
        run1d(2, prog, timeout=5)
    assert isinstance(info.value.failures[0], CollectiveError)
