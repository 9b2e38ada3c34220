"""Product integer planning (paper_2605_11111_b200.plan) — bit-exact vs
integers captured from the reference (tests/golden/plans.json)."""

import math

import pytest
from hypothesis import given
from hypothesis import strategies as hs

from paper_2605_11111_b200 import plan
from paper_2605_11111_b200.errors import DimensionError, ShapeError


def test_default_chunk_kats(plans_golden):
    for extent, members, want in plans_golden["default_chunk"]:
        assert plan.default_chunk(extent, members) == want


def test_default_chunk_rejects_bad_args():
    with pytest.raises(DimensionError):
        plan.default_chunk(-1, 2)
    with pytest.raises(DimensionError):
        plan.default_chunk(4, 0)


@given(extent=hs.integers(0, 10_000), members=hs.integers(1, 64))
def test_default_chunk_properties(extent, members):
    parts = plan.default_chunk(extent, members)
    assert len(parts) == members and sum(parts) == extent and min(parts) >= 0
    c = math.ceil(extent / members) if extent else 0
    nz = [p for p in parts if p]
    assert parts == nz + [0] * (members - len(nz))
    assert all(p == c for p in nz[:-1])


def test_halo_plans_bit_exact_vs_reference(plans_golden):
    ok = errs = 0
    for c in plans_golden["halo_plans"]:
        hp = plan.halo_conv_plan(c["extents"], c["g_in"], c["k"], c["s"], c["p"])
        if "error" in c:
            # the reference failed with a multi-hop HaloError: the plan says so
            v = hp.hop_violations()
            assert v, c
            requester, width, server, extent = v[0]
            assert f"requested halo width {width}" in c["error"]
            assert "single-hop" in c["error"]
            errs += 1
            continue
        assert list(hp.out_extents) == c["out_extents"]
        assert [[m.lw, m.rw] for m in hp.members] == c["widths"]
        assert not hp.hop_violations()
        ok += 1
    assert ok > 100 and errs > 10


def test_left_width_is_always_zero_and_right_bounded():
    for g in range(1, 30):
        for k in (1, 3, 5, 7):
            for s in (1, 2, 3):
                for p in range(0, k // 2 + 2):
                    if (g + 2 * p - k) // s + 1 < 1:
                        continue
                    for r in (1, 2, 3, 5):
                        ext = plan.default_chunk(g, r)
                        hp = plan.halo_conv_plan(ext, g, k, s, p)
                        assert all(m.lw == 0 for m in hp.members)
                        assert all(m.rw <= k - 1 for m in hp.members)
                        assert sum(hp.out_extents) == hp.g_out


def test_cfg_plans():
    assert plan.halo_conv_plan([512, 512], 1024, 3, 1, 1).out_extents == (513, 511)
    hp = plan.halo_conv_plan([32] * 8, 256, 3, 1, 1)
    assert hp.out_extents == (33, 32, 32, 32, 32, 32, 32, 31)
    assert hp.members[0].base == -1 and hp.members[1].base == 0
    hp2 = plan.halo_conv_plan(list(hp.out_extents), 256, 3, 1, 1)
    assert hp2.out_extents == (34, 32, 32, 32, 32, 32, 32, 30)


def test_conv_output_extent_errors():
    with pytest.raises(ShapeError, match="output extent"):
        plan.conv_output_extent(4, 5, 1, 0)


def test_ring_source_order():
    # member i holds member (i - t) mod R's block at step t
    assert [plan.ring_source(1, t, 4) for t in range(4)] == [1, 0, 3, 2]
