"""Dispatch on device tensors: the GPU fallback path (gather -> dense device
op -> default_chunk re-scatter) against the reference's own fallback outputs
(tests/golden/dispatch_cases.npz, made by tests/golden/make_golden.py), and
the reference's device-op trace KATs (pkg/tests/test_dispatch.py:242-283)."""

import json

import numpy as np
import pytest
import torch

from conftest import load_npz, rel_err, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"
CASES = load_npz("dispatch_cases.npz")


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


@pytest.mark.parametrize("i", range(int(CASES["count"])))
def test_fallback_matches_reference_golden(i):
    """Shard shapes, placements and the trace record ("fallback", one
    collective per gathered argument: 3 for sdpa) equal the reference's;
    each rank's block is bit-identical to its default_chunk slice of the
    dense device result and within fp tolerance of the reference's block."""
    import paper_2605_11111_b200 as m

    meta = json.loads(str(CASES[f"f{i}_meta"]))
    op, ext, kext = meta["op"], tuple(meta["ext"]), meta["kext"]
    R = len(ext)
    names = ("q", "k", "v") if op == "sdpa" else ("a", "b")
    ins = {n: torch.tensor(CASES[f"f{i}_{n}"]) for n in names}
    dense = m.DENSE_REFERENCE[op](*(ins[n].to(DEV) for n in names))

    def prog(ctx):
        root = ctx.rank_id == 0
        if op == "sdpa":
            args = [m.scatter_global(ctx, ins["q"] if root else None, (m.Shard(0),), {0: ext})]
            args += [m.scatter_global(ctx, ins[n] if root else None, (m.Shard(0),),
                                      {0: tuple(kext)}) for n in ("k", "v")]
        else:
            args = [m.scatter_global(ctx, ins["a"] if root else None, (m.Shard(0),), {0: ext}),
                    m.replicated(ctx, ins["b"])]
        out = m.dispatch_operation(op, *args)
        lo, hi = out.shard_interval(0)
        return (out.local.cpu(), {str(a): list(e) for a, e in out.shard_shapes.items()},
                [str(p) for p in out.placements], m.trace_lines(ctx)[-1], lo, hi)

    tol = 1e-12 if ins[names[0]].dtype == torch.float64 else 1e-5
    dense_h = dense.cpu()
    for r, (loc, shapes, pl, line, lo, hi) in enumerate(m.spawn_mesh((R,), ("domain",), prog)):
        assert shapes == meta["shapes"]
        assert pl == meta["placements"]
        assert line == meta["trace"]
        assert torch.equal(loc, dense_h[lo:hi])                       # bit-exact re-chunk
        want = CASES[f"f{i}_local{r}"]
        assert tuple(loc.shape) == want.shape
        assert rel_err(to_np(loc), want, 1e-300 if want.size else 1.0) < tol


def test_trace_ring_buffer_is_bounded():
    import paper_2605_11111_b200 as m

    def prog(ctx):
        x = m.replicated(ctx, torch.ones(1, device=DEV))
        for i in range(1100):
            m.dispatch_operation("scale", x, float(i))
        lines = m.trace_lines(ctx)
        assert len(ctx.trace) == 1024 and len(lines) == 1024
        assert lines[0] == "op=scale level=aten_like collectives=0"
        return True

    assert m.spawn_mesh((1,), ("domain",), prog) == [True]


def test_trace_lines_show_collective_costs():
    import paper_2605_11111_b200 as m

    def prog(ctx):
        g = torch.arange(12.0, dtype=torch.float64).reshape(2, 6)
        x = m.scatter_global(ctx, g if ctx.rank_id == 0 else None, (m.Shard(1),))
        m.dispatch_operation("softmax", x, 1)
        m.dispatch_operation("add", x, x)
        return m.trace_lines(ctx)

    for lines in m.spawn_mesh((2,), ("domain",), prog):
        assert lines == ["op=softmax level=aten_like collectives=2",
                         "op=add level=aten_like collectives=0"]
