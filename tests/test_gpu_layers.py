"""SURVEY §8(f) rows on one B200 with R thread-ranks: sharded softmax /
layer norm over uneven (and empty) shards, pointwise + linear ops, ddp
gradient averaging and the ViT block pipeline — against the reference's
own outputs (tests/golden/layer_cases.npz) and the oracle."""

import numpy as np
import pytest
import torch

from conftest import load_npz, rel_err, to_np
from test_oracle import _layer_specs
from oracle import layers as olay

pytestmark = pytest.mark.gpu
DEV = "cuda"
LAYERS = load_npz("layer_cases.npz")
NORM_SPECS, VIT_SPECS = _layer_specs()


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


def dp():
    import paper_2605_11111_b200 as m

    return m


@pytest.mark.parametrize("i", range(len(NORM_SPECS)))
def test_sharded_norm_matches_reference_golden(i):
    m = dp()
    op, shape, sdim, ext, rdim, dt = NORM_SPECS[i]
    x, want = LAYERS[f"n{i}_x"], LAYERS[f"n{i}_y"]

    def prog(ctx):
        xt = torch.tensor(x) if ctx.rank_id == 0 else None
        st = m.scatter_global(ctx, xt, (m.Shard(sdim),), {0: ext})
        before = ctx.collective_count
        y = m.dispatch_operation(op, st, rdim)
        n_coll = ctx.collective_count - before
        assert m.trace_lines(ctx)[-1] == f"op={op} level=aten_like collectives={n_coll}"
        return y.full_tensor(), n_coll, y.shard_shapes

    res = m.spawn_mesh((len(ext),), ("domain",), prog)
    tol = 1e-12 if dt == np.float64 else 1e-5
    assert rel_err(to_np(res[0][0]), want) < tol
    assert res[0][1] == int(LAYERS[f"n{i}_coll"])
    assert res[0][2] == {0: tuple(ext)}


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
def test_dense_norms_large_rows_vs_oracle(dtype):
    """Long reduced dims on the split-partials path (both reduce layouts)."""
    m = dp()
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 70000, 5)) * 2 + 1
    xt = torch.tensor(x).to(dtype).to(DEV)
    xr = to_np(xt).astype(np.float64)
    # fp64: 70000-term sums in a different (chunked) order than NumPy's pairwise
    # sum; E[x^2] - mean^2 turns that ~1e-16*sqrt(n) into ~1e-11 relative
    tol = {torch.float64: 1e-10, torch.float32: 1e-5, torch.bfloat16: 1e-2}[dtype]
    for dim in (1, 2, 0):
        assert rel_err(to_np(m.dense_layer_norm(xt, dim)), olay.layer_norm(xr, dim)) < tol
        assert rel_err(to_np(m.dense_softmax(xt, dim)), olay.softmax(xr, dim)) < tol


def test_norm_errors():
    m = dp()

    def prog(ctx):
        st = m.scatter_global(ctx, torch.zeros(4, 0) if ctx.rank_id == 0 else None,
                              (m.Shard(0),))
        with pytest.raises(m.DegenerateInputError, match="zero-extent dim 1"):
            m.dispatch_operation("softmax", st, 1)
        with pytest.raises(m.DegenerateInputError, match="zero-extent dim 1"):
            m.dispatch_operation("layer_norm", st, -1)
        with pytest.raises(m.DimensionError, match="out of range"):
            m.dispatch_operation("layer_norm", st, 2)
        return True

    assert all(m.spawn_mesh((2,), ("domain",), prog))


def test_elementwise_and_linear():
    m = dp()
    rng = np.random.default_rng(2)
    a = rng.standard_normal((9, 6)).astype(np.float32)
    b = rng.standard_normal((9, 6)).astype(np.float32)
    w = rng.standard_normal((4, 6)).astype(np.float32)
    bias = rng.standard_normal(4).astype(np.float32)

    def prog(ctx):
        root = ctx.rank_id == 0
        sa = m.scatter_global(ctx, torch.tensor(a) if root else None, (m.Shard(0),), {0: (5, 0, 4)})
        sb = m.scatter_global(ctx, torch.tensor(b) if root else None, (m.Shard(0),), {0: (5, 0, 4)})
        before = ctx.collective_count
        add = m.dispatch_operation("add", sa, sb)
        mul = m.dispatch_operation("mul", sa, sb)
        sc = m.dispatch_operation("scale", sa, 2.5)
        adds = m.dispatch_operation("add", sa, 1.25)
        lin = m.dispatch_operation("linear", sa, torch.tensor(w), torch.tensor(bias))
        assert ctx.collective_count == before
        sc2 = m.scatter_global(ctx, torch.tensor(b) if root else None, (m.Shard(0),))
        with pytest.raises(m.MetadataError, match="operand layouts disagree"):
            m.dispatch_operation("add", sa, sc2)
        with pytest.raises(m.DimensionError, match="scale expects a scalar"):
            m.dispatch_operation("scale", sa, torch.ones(2, device=DEV))
        with pytest.raises(m.UnsupportedConfigError, match="contraction dim"):
            st1 = m.scatter_global(ctx, torch.tensor(a) if root else None, (m.Shard(1),))
            m.dispatch_operation("linear", st1, torch.tensor(w), torch.tensor(bias))
        return [t.full_tensor() for t in (add, mul, sc, adds, lin)]

    add, mul, sc, adds, lin = m.spawn_mesh((3,), ("domain",), prog)[0]
    assert np.array_equal(to_np(add), a + b)
    assert np.array_equal(to_np(mul), a * b)
    assert np.array_equal(to_np(sc), a * np.float32(2.5))
    assert np.array_equal(to_np(adds), a + np.float32(1.25))
    assert rel_err(to_np(lin), a.astype(np.float64) @ w.T.astype(np.float64) + bias) < 1e-5


def test_ddp_allreduce_grads_matches_reference():
    m = dp()
    g = LAYERS["ddp_grads"]

    def prog(ctx):
        grads = {"w": torch.tensor(g[ctx.rank_id], device=DEV),
                 "b": torch.tensor(g[ctx.rank_id][0], device=DEV)}
        out = m.ddp_allreduce_grads(ctx.axis_group("data"), grads)
        lst = m.ddp_allreduce_grads(ctx.axis_group("data"), (grads["w"],))
        assert isinstance(lst, tuple)
        return out

    res = m.spawn_mesh((3,), ("data",), prog)
    for r in res:
        assert rel_err(to_np(r["w"]), LAYERS["ddp_w"]) < 1e-15
        assert rel_err(to_np(r["b"]), LAYERS["ddp_b"]) < 1e-15


def test_image_to_sequence_bitwise():
    m = dp()
    x = np.arange(3 * 7 * 5, dtype=np.float32).reshape(3, 7, 5)

    def prog(ctx):
        st = m.scatter_global(ctx, torch.tensor(x) if ctx.rank_id == 0 else None,
                              (m.Shard(1),), {0: (3, 0, 4)})
        seq = m.image_to_sequence(st)
        return seq.full_tensor(), seq.shard_shapes, seq.placements

    full, shapes, pl = m.spawn_mesh((3,), ("domain",), prog)[0]
    assert np.array_equal(to_np(full), np.transpose(x, (1, 2, 0)).reshape(-1, 3))
    assert shapes == {0: (15, 0, 20)} and pl == (m.Shard(0),)


@pytest.mark.parametrize("i", range(len(VIT_SPECS)))
def test_vit_block_pipeline_matches_reference(i):
    """vit_block_pipeline (halo-conv tokenizer, sequence-sharded layer norms,
    one all-heads ring per layer) vs the reference's own sharded run and its
    dense twin; same weights bit for bit, same activation-ledger bytes."""
    m = dp()
    img, ext, kw, dt = VIT_SPECS[i]
    cfg = m.VitConfig(image_channels=img[0], **{k: v for k, v in kw.items()
                                                if k != "image_channels"})
    tdt = torch.float64 if dt == np.float64 else torch.float32
    weights = m.make_vit_weights(cfg, seed=i, dtype=tdt, device=DEV)
    ow = olay.vit_weights(cfg.embed_dim, img[0], cfg.patch, cfg.n_layers, cfg.mlp_hidden,
                          seed=i, dtype=dt)
    assert all(np.array_equal(to_np(weights[k]), ow[k]) for k in ow)
    x = LAYERS[f"v{i}_x"]

    def prog(ctx):
        st = m.scatter_global(ctx, torch.tensor(x) if ctx.rank_id == 0 else None,
                              (m.Shard(1),), {0: ext})
        led = m.ActivationLedger()
        seq = m.vit_block_pipeline(st, cfg, weights, ledger=led)
        return seq.full_tensor(), led.peak_bytes, list(seq.shard_shapes[0])

    res = m.spawn_mesh((len(ext),), ("domain",), prog)
    tol = 1e-10 if dt == np.float64 else 1e-4
    assert rel_err(to_np(res[0][0]), LAYERS[f"v{i}_y"]) < tol
    assert res[0][2] == list(LAYERS[f"v{i}_shapes"])
    assert [r[1] for r in res] == list(LAYERS[f"v{i}_ledger"])
    dense = m.vit_block_pipeline_dense(torch.tensor(x, device=DEV), cfg, weights)
    assert rel_err(to_np(dense), LAYERS[f"v{i}_dense"]) < tol
