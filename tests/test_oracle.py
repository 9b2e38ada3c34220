"""The oracle pinned before it is trusted: against the reference's golden
outputs (bit-exact for integers and forward conv), nested loops, and
central finite differences for the restated backward."""

import json
import math

import numpy as np
import pytest

from conftest import load_npz, rel_err
from oracle import attention as oatt
from oracle import conv as oconv
from oracle import plan as oplan
from oracle import sharding as osh


def test_default_chunk_kats(plans_golden):
    for extent, members, want in plans_golden["default_chunk"]:
        assert oplan.default_chunk(extent, members) == want


def test_member_plans_match_reference_capture(plans_golden):
    """Ints captured from the reference's own halo_exchange calls."""
    checked = 0
    for c in plans_golden["halo_plans"]:
        if "error" in c:
            continue
        plans = oplan.member_plans(c["extents"], c["g_in"], c["k"], c["s"], c["p"])
        assert [p[1] - p[0] for p in plans] == c["out_extents"]
        assert [[p[4], p[5]] for p in plans] == c["widths"]
        checked += 1
    assert checked > 100


def test_conv_restatement_bitwise_vs_reference_outputs():
    d = load_npz("conv_cases.npz")
    for i in range(int(d["count"])):
        meta = json.loads(str(d[f"c{i}_meta"]))
        s = meta["stride"] if isinstance(meta["stride"], int) else tuple(meta["stride"])
        p = meta["padding"] if isinstance(meta["padding"], int) else tuple(meta["padding"])
        got = oconv.conv(d[f"c{i}_x"], d[f"c{i}_w"], s, p)
        assert np.array_equal(got, d[f"c{i}_y"])  # bitwise: same einsum construction
        outs, ext = oconv.halo_conv_members(d[f"c{i}_x"], d[f"c{i}_w"], meta["extents"],
                                            meta["dim"], s, p)
        assert ext == meta["out_extents"]
        assert np.array_equal(np.concatenate(outs, axis=meta["dim"]), d[f"c{i}_y"])


def _conv_loops(x, w, s, p):
    """Nested-loop conv, float64 (style of pkg/tests/test_dense.py:35-61)."""
    n = w.ndim - 2
    xp = np.pad(x, [(0, 0), (0, 0)] + [(p, p)] * n)
    outs = [(g + 2 * p - k) // s + 1 for g, k in zip(x.shape[2:], w.shape[2:])]
    y = np.zeros((x.shape[0], w.shape[0]) + tuple(outs))
    for b in range(x.shape[0]):
        for co in range(w.shape[0]):
            for o in np.ndindex(*outs):
                acc = 0.0
                for ci in range(x.shape[1]):
                    for t in np.ndindex(*w.shape[2:]):
                        idx = tuple(oo * s + tt for oo, tt in zip(o, t))
                        acc += xp[(b, ci) + idx] * w[(co, ci) + t]
                y[(b, co) + o] = acc
    return y


@pytest.mark.parametrize("n,s,p", [(1, 2, 1), (2, 1, 1), (3, 1, 1), (3, 2, 0)])
def test_conv_nd_against_nested_loops(n, s, p):
    rng = np.random.default_rng(n * 10 + s)
    x = rng.standard_normal((2, 2) + (5,) * n)
    w = rng.standard_normal((3, 2) + (3,) * n)
    assert np.allclose(oconv.conv(x, w, s, p), _conv_loops(x, w, s, p), atol=1e-12)


@pytest.mark.parametrize("n,s,p", [(1, 2, 1), (2, 1, 1), (2, 3, 2), (3, 1, 1), (3, 2, 0)])
def test_conv_fast_matches_reference_einsum(n, s, p):
    """The BLAS tap-sum oracle (large parity cases) equals the reference's
    einsum restatement to fp64 rounding."""
    rng = np.random.default_rng(n * 7 + s + p)
    x = rng.standard_normal((2, 3) + (7,) * n)
    w = rng.standard_normal((4, 3) + (3,) * n)
    want = oconv.conv(x, w, s, p)
    got = oconv.conv_fast(x, w, s, p)
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("n,s,p", [(1, 1, 1), (2, 2, 1), (3, 1, 1)])
def test_conv_grads_central_differences(n, s, p):
    rng = np.random.default_rng(5 + n)
    x = rng.standard_normal((1, 2) + (6,) * n)
    w = rng.standard_normal((2, 2) + (3,) * n)
    dy = rng.standard_normal(oconv.conv(x, w, s, p).shape)
    dx, dw = oconv.conv_grads(x, w, dy, s, p)
    f = lambda xx, ww: float((oconv.conv(xx, ww, s, p) * dy).sum())  # noqa: E731
    eps = 1e-6
    for _ in range(6):
        i = tuple(int(rng.integers(0, e)) for e in x.shape)
        xp, xm = x.copy(), x.copy()
        xp[i] += eps
        xm[i] -= eps
        assert abs((f(xp, w) - f(xm, w)) / (2 * eps) - dx[i]) < 1e-6
        j = tuple(int(rng.integers(0, e)) for e in w.shape)
        wp, wm = w.copy(), w.copy()
        wp[j] += eps
        wm[j] -= eps
        assert abs((f(x, wp) - f(x, wm)) / (2 * eps) - dw[j]) < 1e-6


def test_sharded_conv_backward_adjoint_is_global_gradient():
    """Restated A9 adjoint: per-member dgrad over the virtual block plus the
    reverse halo into member m+1 equals the global dx; member wgrads sum
    to the global dw."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1, 3, 14, 5))
    w = rng.standard_normal((2, 3, 3, 3))
    ext = [4, 0, 6, 4]
    dy = rng.standard_normal(oconv.conv(x, w, 1, 1).shape)
    dx_ref, dw_ref = oconv.conv_grads(x, w, dy, 1, 1)
    plans = oplan.member_plans(ext, 14, 3, 1, 1)
    bounds = np.concatenate([[0], np.cumsum(ext)]).astype(int)
    dx = np.zeros_like(x)
    dw = np.zeros_like(w)
    ob = np.concatenate([[0], np.cumsum([p[1] - p[0] for p in plans])]).astype(int)
    for m, (j_lo, j_hi, w_min, w_max, lw, rw) in enumerate(plans):
        if j_hi == j_lo:
            continue
        lo, hi = max(w_min, 0), min(w_max, 14)
        blk = x[:, :, lo:hi]
        pad = (max(0, -w_min), max(0, w_max - 14))
        blk = np.pad(blk, [(0, 0), (0, 0), pad, (0, 0)])
        gx, gw = oconv.conv_grads(blk, w, dy[:, :, ob[m]:ob[m + 1]], (1, 1), (0, 1))
        gx = gx[:, :, pad[0]:gx.shape[2] - pad[1]]
        dx[:, :, lo:hi] += gx  # rows >= bounds[m+1] are member m+1's (single hop)
        assert hi <= bounds[m + 1] + rw
        dw += gw
    assert rel_err(dx, dx_ref) < 1e-13
    assert rel_err(dw, dw_ref) < 1e-13


def test_ring_restatement_vs_reference_outputs():
    d = load_npz("ring_cases.npz")
    for i in range(int(d["count"])):
        q, k, v, o = (d[f"r{i}_{n}"] for n in ("q", "k", "v", "o"))
        outs = oatt.ring_members(q, k, v, list(d[f"r{i}_qe"]), list(d[f"r{i}_ke"]))
        got = np.concatenate(outs, axis=0)
        tol = 1e-13 if q.dtype == np.float64 else 1e-6
        assert rel_err(got, o) < tol
        assert rel_err(oatt.sdpa(q, k, v), o) < (1e-12 if q.dtype == np.float64 else 1e-5)


def test_ring_state_prefix_invariant():
    """pkg/tests/test_ops.py:240-268 restated against the oracle state."""
    rng = np.random.default_rng(500)
    st = oatt.RingState(3, 2)
    ss, vs = np.zeros((3, 0)), np.zeros((0, 2))
    for w in (2, 0, 3, 1):
        s = rng.standard_normal((3, w)) * 4
        v = rng.standard_normal((w, 2))
        st.update(s, v)
        ss, vs = np.concatenate([ss, s], 1), np.concatenate([vs, v], 0)
        if ss.shape[1]:
            assert np.allclose(st.output(), oatt.softmax64(ss) @ vs, atol=1e-12)


def test_sdpa_grads_central_differences():
    rng = np.random.default_rng(3)
    q, k, v, do = (rng.standard_normal(s) for s in ((4, 2, 3), (5, 2, 3), (5, 2, 3), (4, 2, 3)))
    dq, dk, dv = oatt.sdpa_grads(q, k, v, do)
    f = lambda a, b, c: float((oatt.sdpa(a, b, c) * do).sum())  # noqa: E731
    eps = 1e-6
    for arr, grad, pos in ((q, dq, 0), (k, dk, 1), (v, dv, 2)):
        for _ in range(5):
            i = tuple(int(rng.integers(0, e)) for e in arr.shape)
            ap, am = arr.copy(), arr.copy()
            ap[i] += eps
            am[i] -= eps
            args_p = [q, k, v]
            args_m = [q, k, v]
            args_p[pos], args_m[pos] = ap, am
            fd = (f(*args_p) - f(*args_m)) / (2 * eps)
            assert abs(fd - grad[i]) < 1e-6


def test_redistribute_restatement_vs_reference_blocks():
    d = load_npz("redist_cases.npz")
    for i in range(int(d["count"])):
        meta = json.loads(str(d[f"d{i}_meta"]))
        if len(meta["mesh"]) != 1:
            continue
        g = d[f"d{i}_g"]
        r = meta["mesh"][0]
        new = meta["new"][0]
        if new == "Replicate":
            for rank in range(r):
                assert np.array_equal(d[f"d{i}_local{rank}"], g)
            continue
        blocks, ext = osh.reshard_1d(g, None, int(new[6:-1]), r)
        assert list(ext) == meta["out_shapes"]["0"]
        for rank in range(r):
            assert np.array_equal(blocks[rank], d[f"d{i}_local{rank}"])
    assert math.isfinite(1.0)


# ---- §8(f): normalisations and the ViT pipeline (tests/golden/layer_cases.npz)

def _layer_specs():
    import importlib.util
    import os
    from conftest import GOLDEN

    spec = importlib.util.spec_from_file_location("_mk", os.path.join(GOLDEN, "make_golden.py"))
    src = open(os.path.join(GOLDEN, "make_golden.py")).read()
    # the spec tables only (the module itself imports the reference)
    ns = {"np": np}
    start = src.index("NORM_SPECS = [")
    end = src.index("def make_layer_cases")
    exec(src[start:end], ns)
    return ns["NORM_SPECS"], ns["VIT_SPECS"]


def test_norm_restatement_vs_reference_outputs():
    from oracle import layers as olay

    d = load_npz("layer_cases.npz")
    norm_specs, _ = _layer_specs()
    for i, (op, shape, sdim, ext, rdim, dt) in enumerate(norm_specs):
        x, want = d[f"n{i}_x"], d[f"n{i}_y"]
        got = olay.softmax(x, rdim) if op == "softmax" else olay.layer_norm(x, rdim)
        tol = 1e-12 if dt == np.float64 else 1e-6
        assert rel_err(got, want) < tol, (i, op)
        # collectives: 2 for a sharded softmax, 1 for a sharded layer norm, 0 local
        sharded = (rdim % len(shape)) == sdim
        assert int(d[f"n{i}_coll"]) == ((2 if op == "softmax" else 1) if sharded else 0)


def test_vit_restatement_vs_reference_outputs():
    from oracle import layers as olay

    d = load_npz("layer_cases.npz")
    _, vit_specs = _layer_specs()
    for i, (img, ext, kw, dt) in enumerate(vit_specs):
        cfg = dict(dict(embed_dim=64, n_layers=16, n_heads=4, mlp_ratio=4), **kw)
        w = olay.vit_weights(cfg["embed_dim"], img[0], 5, cfg["n_layers"],
                             cfg["embed_dim"] * cfg["mlp_ratio"], seed=i, dtype=dt)
        got = olay.vit_dense(d[f"v{i}_x"], w, 5, cfg["n_layers"], cfg["n_heads"])
        tol = 1e-10 if dt == np.float64 else 1e-4
        assert rel_err(got, d[f"v{i}_dense"]) < tol
        assert rel_err(got, d[f"v{i}_y"]) < tol   # the sharded reference run agrees


def test_ddp_mean_golden():
    d = load_npz("layer_cases.npz")
    g = d["ddp_grads"]
    assert rel_err(d["ddp_w"], g.sum(0) / 3) < 1e-15
    assert rel_err(d["ddp_b"], g[:, 0].sum(0) / 3) < 1e-15


def test_stack_window_matches_full_stack():
    """The windowed two-layer oracle (full-size conv parity on slabs) equals
    the same box of the full computation, borders included, for the forward
    and for the input gradient through transposed-flipped weights."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 3, 9, 8, 10))
    w1 = rng.standard_normal((4, 3, 3, 3, 3))
    w2 = rng.standard_normal((2, 4, 3, 3, 3))
    full = oconv.conv(oconv.conv(x, w1, 1, 1), w2, 1, 1)
    for lo, hi in (((0, 0, 0), (3, 4, 5)), ((4, 2, 6), (9, 8, 10)), ((2, 3, 1), (6, 5, 7))):
        got = oconv.stack_window(x, [w1, w2], lo, hi)
        want = full[:, :, lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
        assert np.abs(got - want).max() < 1e-10 * np.abs(want).max()
    dy = rng.standard_normal(full.shape)
    y1 = oconv.conv(x, w1, 1, 1)
    dy1, _ = oconv.conv_grads(y1, w2, dy, 1, 1)
    dx, _ = oconv.conv_grads(x, w1, dy1, 1, 1)
    ws_t = [oconv.transposed_flipped(w2), oconv.transposed_flipped(w1)]
    got = oconv.stack_window(dy, ws_t, (3, 0, 2), (9, 8, 7))
    assert np.abs(got - dx[:, :, 3:9, 0:8, 2:7]).max() < 1e-10 * np.abs(dx).max()


def test_head_slab_matches_dense_grads():
    from oracle import attention as oatt

    rng = np.random.default_rng(12)
    S, d = 300, 16
    q, k, v, do = (rng.standard_normal((S, d)) for _ in range(4))
    o = oatt.sdpa(q, k, v)
    dq, dk, dv = oatt.sdpa_grads(q, k, v, do)
    rows, keys = slice(100, 164), slice(10, 60)
    so, sdq, sdk, sdv = oatt.head_slab(q, k, v, do, rows, keys, chunk=64)
    assert np.abs(so - o[rows]).max() < 1e-12
    assert np.abs(sdq - dq[rows]).max() < 1e-12
    assert np.abs(sdk - dk[keys]).max() < 1e-5     # row stats from fp32 score chunks
    assert np.abs(sdv - dv[keys]).max() < 1e-5
