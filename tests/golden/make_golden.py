"""Generate the golden fixtures by running the REAL reference (`domainpar`
from /root/reference/pkg/src) in this container.  The reference cannot
travel to the GPU box, so its outputs are committed here as small fixtures:

  plans.json        per-member (out_extent, left_width, right_width) of
                    halo_conv captured from the reference's own halo_exchange
                    calls, for KAT and random configurations; default_chunk
                    KATs; debug_line strings
  conv_cases.npz    halo_conv inputs and the reference's gathered outputs
  ring_cases.npz    ring_attention inputs and the reference's outputs
  redist_cases.npz  redistribute inputs and the reference's per-rank blocks
  layer_cases.npz   sharded_softmax / sharded_layer_norm (uneven shards),
                    ddp_allreduce_grads and vit_block_pipeline outputs
  dispatch_cases.npz  the fallback path (gather -> dense -> default_chunk
                    re-scatter) on sdpa / matmul: blocks, shapes, trace

Run:  python tests/golden/make_golden.py [core|layers|dispatch]   (needs /root/reference)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import domainpar  # noqa: E402
from domainpar import ops as rops  # noqa: E402
from domainpar.mesh import spawn_mesh  # noqa: E402
from domainpar.sharding import (Replicate, Shard, ShardTensor, default_chunk, replicated,  # noqa: E402
                                redistribute, scatter_global)
from domainpar.verify import random_partition  # noqa: E402


def capture_plan(extents, g_in, k, s, p):
    """Run the reference halo_conv on a 1-channel 1-D input and record what
    each rank asked halo_exchange for, plus the output shard shapes."""
    calls = {}
    real = rops.halo_exchange

    def spy(group, local, dim, lw, rw):
        calls[group.ctx.rank_id] = (int(lw), int(rw))
        return real(group, local, dim, lw, rw)

    x = np.arange(g_in, dtype=np.float64).reshape(1, g_in)
    w = np.ones((1, 1, k))

    def prog(ctx):
        st = ShardTensor(x[:, sum(extents[:ctx.rank_id]):sum(extents[:ctx.rank_id + 1])],
                         (1, g_in), ctx, (Shard(1),), {0: tuple(extents)})
        out = rops.halo_conv(st, w, stride=s, padding=p)
        return out.shard_shapes[0]

    rops.halo_exchange = spy
    try:
        res = spawn_mesh((len(extents),), ("domain",), prog)
        err = None
    except Exception as e:  # noqa: BLE001 - recorded as an expected failure
        res, err = None, str(e)
    finally:
        rops.halo_exchange = real
    if err is not None:
        return {"extents": extents, "g_in": g_in, "k": k, "s": s, "p": p, "error": err}
    return {"extents": extents, "g_in": g_in, "k": k, "s": s, "p": p,
            "out_extents": list(res[0]), "widths": [list(calls[r]) for r in range(len(extents))]}


def make_plans():
    rng = np.random.default_rng(2605)
    cases = []
    kats = [([512, 512], 1024, 3, 1, 1),            # cfg1 -> (513, 511)
            ([32] * 8, 256, 3, 1, 1),               # cfg2 layer 1
            ([33] + [32] * 6 + [31], 256, 3, 1, 1),  # cfg2 layer 2 (drifted)
            ([5, 5], 10, 3, 2, 1),                  # acceptance (3, 2)
            ([4, 5], 9, 1, 3, 0),                   # (2, 1)
            ([3, 0, 2], 5, 1, 1, 0),                # empty shard
            ([5, 4, 3], 12, 3, 2, 1),
            ([4, 4], 8, 5, 1, 4),
            ([3, 1, 2], 6, 3, 1, 0)]                # multi-hop -> HaloError
    for e, g, k, s, p in kats:
        cases.append(capture_plan(list(e), g, k, s, p))
    while len(cases) < 260:
        r = int(rng.integers(1, 9))
        k = int(rng.choice([1, 3, 5, 7]))
        s = int(rng.integers(1, 4))
        p = int(rng.integers(0, k // 2 + 2))
        g = int(rng.integers(max(1, k - 2 * p), 40))
        if (g + 2 * p - k) // s + 1 < 1:
            continue
        ext = [int(v) for v in random_partition(rng, g, r, min_part=0)]
        cases.append(capture_plan(ext, g, k, s, p))
    chunks = [[e, m, default_chunk(e, m)] for e, m in
              [(10, 4), (5, 4), (0, 3), (7, 1), (3, 5), (8, 2), (17, 5), (9, 4), (6, 4),
               (1024, 2), (256, 8), (65536, 8), (65536, 3)]]

    def dl(ctx):
        root = ctx.rank_id == 0
        st = scatter_global(ctx, np.zeros((5, 3)) if root else None, (Shard(0),), {0: (3, 0, 2)})
        rep = replicated(ctx, np.arange(4.0))
        return st.debug_line(), rep.debug_line()

    lines = spawn_mesh((3,), ("domain",), dl)

    def dl2(ctx):
        root = ctx.rank_id == 0
        st = scatter_global(ctx, np.zeros((4, 6)) if root else None, (Shard(0), Shard(1)))
        return st.debug_line()

    lines2 = spawn_mesh((2, 3), ("a", "b"), dl2)
    return {"halo_plans": cases, "default_chunk": chunks, "debug_lines": lines,
            "debug_lines_2d": lines2}


def make_conv_cases():
    rng = np.random.default_rng(11)
    specs = [
        # (global shape, kernel shape tail, stride, padding, shard dim, extents, dtype)
        ((2, 10), (3,), 2, 1, 1, (5, 5), np.float64),
        ((1, 5), (1,), 1, 0, 1, (3, 0, 2), np.float32),
        ((2, 3, 12, 7), (3, 5), (2, 1), (1, 2), 2, (5, 4, 3), np.float64),
        ((1, 9), (1,), 3, 0, 1, (4, 5), np.float64),
        ((2, 8), (5,), 1, 4, 1, (4, 4), np.float64),
        ((1, 4, 16, 16), (3, 3), 1, 1, 2, (6, 5, 5), np.float32),
        ((1, 4, 16, 16), (3, 3), 1, 1, 3, (3, 7, 6), np.float32),
        ((2, 3, 20, 9), (5, 3), (1, 2), (2, 1), 2, (4, 7, 4, 5), np.float64),
        ((3, 33), (3,), 1, 1, 1, (11, 11, 11), np.float32),
        ((1, 8, 32, 24), (3, 3), 1, 1, 2, (8, 8, 8, 8), np.float32),
        ((1, 8, 32, 24), (3, 3), 2, 1, 2, (10, 9, 7, 6), np.float32),
        ((2, 16, 18, 10), (3, 3), 1, 0, 2, (7, 6, 5), np.float64),
    ]
    out = {}
    for i, (shape, ktail, stride, pad, dim, ext, dt) in enumerate(specs):
        n = len(ktail)
        cin = shape[-n - 1]
        cout = int(rng.integers(1, 5)) if cin < 8 else 8
        x = rng.standard_normal(shape).astype(dt)
        w = (rng.standard_normal((cout, cin) + ktail) * 0.5).astype(dt)

        def prog(ctx, x=x, w=w, dim=dim, ext=ext, stride=stride, pad=pad):
            st = scatter_global(ctx, x if ctx.rank_id == 0 else None, (Shard(dim),), {0: ext})
            res = rops.halo_conv(st, w, stride=stride, padding=pad)
            return res.full_tensor(), res.shard_shapes[0]

        res = spawn_mesh((len(ext),), ("domain",), prog)
        full, shapes = res[0]
        dense = domainpar.conv(x, w, stride=stride, padding=pad)
        assert np.array_equal(full, dense), i
        out[f"c{i}_x"] = x
        out[f"c{i}_w"] = w
        out[f"c{i}_y"] = full
        out[f"c{i}_meta"] = np.array(json.dumps({"stride": stride, "padding": pad, "dim": dim,
                                                 "extents": list(ext),
                                                 "out_extents": list(shapes)}))
    out["count"] = np.array(len(specs))
    return out


def make_ring_cases():
    rng = np.random.default_rng(7)
    specs = [
        (5, 11, 6, (2, 0, 3, 0), (4, 0, 5, 2), np.float64),
        (4, 6, 4, (2, 2), (3, 3), np.float32),
        (12, 12, 16, (5, 0, 4, 3), (5, 0, 4, 3), np.float64),
        (12, 12, 16, (5, 0, 4, 3), (5, 0, 4, 3), np.float32),
        (19, 17, 8, (3, 5, 4, 7), (9, 0, 0, 8), np.float64),
        (64, 96, 32, (16, 16, 16, 16), (24, 24, 24, 24), np.float32),
        (40, 40, 64, (5,) * 8, (5,) * 8, np.float32),
    ]
    out = {}
    for i, (sq, sk, d, qe, ke, dt) in enumerate(specs):
        q = rng.standard_normal((sq, d)).astype(dt)
        k = rng.standard_normal((sk, d)).astype(dt)
        v = rng.standard_normal((sk, d)).astype(dt)
        if i == 1:
            q = q * 100
            k = k * 100

        def prog(ctx, q=q, k=k, v=v, qe=qe, ke=ke):
            root = ctx.rank_id == 0
            qs = scatter_global(ctx, q if root else None, (Shard(0),), {0: qe})
            ks = scatter_global(ctx, k if root else None, (Shard(0),), {0: ke})
            vs = scatter_global(ctx, v if root else None, (Shard(0),), {0: ke})
            return rops.ring_attention(qs, ks, vs).full_tensor()

        full = spawn_mesh((len(qe),), ("domain",), prog)[0]
        out[f"r{i}_q"], out[f"r{i}_k"], out[f"r{i}_v"], out[f"r{i}_o"] = q, k, v, full
        out[f"r{i}_qe"] = np.array(qe)
        out[f"r{i}_ke"] = np.array(ke)
    out["count"] = np.array(len(specs))
    return out


def make_redist_cases():
    rng = np.random.default_rng(3)
    out = {}
    cases = []
    for r in (2, 3, 4, 5):
        n = 13 + r
        ext = tuple(int(v) for v in random_partition(rng, n, r, min_part=0))
        cases.append(((n, n + 3), (Shard(0),), (Shard(1),), {0: ext}, (r,)))
        cases.append(((n, n + 3), (Shard(0),), (Replicate(),), {0: ext}, (r,)))
        cases.append(((n + 1, n), (Shard(1),), (Shard(0),), None, (r,)))
    cases.append(((6, 8), (Shard(0), Shard(1)), (Shard(1), Shard(0)), None, (2, 2)))
    cases.append(((6, 8), (Shard(0), Replicate()), (Shard(0), Shard(1)), {0: (5, 1)}, (2, 3)))
    cases.append(((4, 3, 5), (Shard(2),), (Shard(0),), {0: (0, 5, 0)}, (3,)))
    for i, (shape, old, new, shapes, mesh) in enumerate(cases):
        g = rng.standard_normal(shape).astype(np.float32)
        names = ("domain",) if len(mesh) == 1 else ("a", "b")

        def prog(ctx, g=g, old=old, new=new, shapes=shapes):
            st = scatter_global(ctx, g if ctx.rank_id == 0 else None, old, shapes)
            r2 = redistribute(st, new)
            return r2.local, {int(a): list(v) for a, v in r2.shard_shapes.items()}

        res = spawn_mesh(mesh, names, prog)
        out[f"d{i}_g"] = g
        for rank, (loc, sh) in enumerate(res):
            out[f"d{i}_local{rank}"] = loc
        meta = {"mesh": list(mesh), "old": [repr(p) for p in old], "new": [repr(p) for p in new],
                "shapes": None if shapes is None else {str(a): list(v) for a, v in shapes.items()},
                "out_shapes": res[0][1]}
        out[f"d{i}_meta"] = np.array(json.dumps(meta))
    out["count"] = np.array(len(cases))
    return out


NORM_SPECS = [
    # op, global shape, sharded dim, extents along it, reduce dim, dtype
    ("softmax", (11, 6), 0, (5, 0, 4, 2), 0, np.float64),
    ("softmax", (11, 6), 0, (5, 0, 4, 2), 1, np.float64),
    ("softmax", (7, 9, 4), 1, (2, 4, 3), 1, np.float32),
    ("softmax", (300, 3), 0, (100, 37, 163), 0, np.float32),
    ("layer_norm", (11, 6), 0, (5, 0, 4, 2), 0, np.float64),
    ("layer_norm", (11, 6), 0, (5, 0, 4, 2), 1, np.float64),
    ("layer_norm", (7, 9, 4), 1, (2, 4, 3), 1, np.float32),
    ("layer_norm", (5, 1000), 1, (400, 0, 600), 1, np.float32),
    ("layer_norm", (12, 8), 0, (6, 6), -2, np.float32),
]

VIT_SPECS = [
    # image (c, h, w), extents along h, config kwargs, dtype
    ((3, 20, 15), (10, 10), dict(embed_dim=16, n_layers=2, n_heads=2, mlp_ratio=2), np.float64),
    ((3, 25, 10), (10, 5, 10), dict(embed_dim=16, n_layers=2, n_heads=4, mlp_ratio=2),
     np.float64),
    ((2, 30, 20), (15, 15), dict(image_channels=2, embed_dim=32, n_layers=1, n_heads=2,
                                 mlp_ratio=4), np.float32),
]


def make_layer_cases():
    """sharded_softmax / sharded_layer_norm over uneven shards, ddp averaging
    and the ViT block pipeline, from the reference (domainpar/ops.py)."""
    rng = np.random.default_rng(11)
    out = {}
    for i, (op, shape, sdim, ext, rdim, dt) in enumerate(NORM_SPECS):
        g = (rng.standard_normal(shape) * 3).astype(dt)
        fn = rops.sharded_softmax if op == "softmax" else rops.sharded_layer_norm

        def prog(ctx, g=g, sdim=sdim, ext=ext, rdim=rdim, fn=fn):
            pl = tuple(Shard(sdim) if a == 0 else Replicate() for a in range(1))
            st = scatter_global(ctx, g if ctx.rank_id == 0 else None, pl, {0: ext})
            before = ctx.collective_count
            y = fn(st, rdim)
            n_coll = ctx.collective_count - before
            return y.full_tensor(), n_coll

        res = spawn_mesh((len(ext),), ("domain",), prog)
        out[f"n{i}_x"], out[f"n{i}_y"] = g, res[0][0]
        out[f"n{i}_coll"] = np.array(res[0][1])
    out["n_count"] = np.array(len(NORM_SPECS))
    # ddp_allreduce_grads over 3 ranks: per-rank grads, the group mean
    grads = [rng.standard_normal((4, 5)) for _ in range(3)]

    def dprog(ctx):
        g = {"w": grads[ctx.rank_id], "b": grads[ctx.rank_id][0]}
        return rops.ddp_allreduce_grads(ctx.axis_group("data"), g)

    dres = spawn_mesh((3,), ("data",), dprog)
    out["ddp_grads"] = np.stack(grads)
    out["ddp_w"], out["ddp_b"] = dres[0]["w"], dres[0]["b"]
    for i, (img, ext, kw, dt) in enumerate(VIT_SPECS):
        cfg = rops.VitConfig(image_channels=img[0], **{k: v for k, v in kw.items()
                                                       if k != "image_channels"})
        weights = rops.make_vit_weights(cfg, seed=i, dtype=dt)
        x = rng.standard_normal(img).astype(dt)

        def vprog(ctx, x=x, ext=ext, cfg=cfg, weights=weights):
            st = scatter_global(ctx, x if ctx.rank_id == 0 else None, (Shard(1),), {0: ext})
            from domainpar.memory import ActivationLedger
            led = ActivationLedger()
            seq = rops.vit_block_pipeline(st, cfg, weights, ledger=led)
            return seq.full_tensor(), led.peak_bytes, list(seq.shard_shapes[0])

        res = spawn_mesh((len(ext),), ("domain",), vprog)
        dense = rops.vit_block_pipeline_dense(x, cfg, weights)
        out[f"v{i}_x"], out[f"v{i}_y"], out[f"v{i}_dense"] = x, res[0][0], dense
        out[f"v{i}_ledger"] = np.array([r[1] for r in res])
        out[f"v{i}_shapes"] = np.array(res[0][2])
    out["v_count"] = np.array(len(VIT_SPECS))
    return out


DISPATCH_SPECS = [
    # (op, q/a extents, k/v extents or None, dtype)
    ("sdpa", (5, 0, 4, 3), (2, 6, 0, 4), "float64"),
    ("sdpa", (3, 3, 3, 3), (4, 4, 2, 2), "float32"),
    ("matmul", (4, 1, 0, 3), None, "float64"),
]


def make_dispatch_cases():
    """The reference's GPU-less fallback path (dispatch.py:156-201) on ops
    with no sharded handler: per-rank blocks, shard shapes, placements and
    the trace record (level "fallback", collectives = gathers)."""
    from domainpar.dispatch import dispatch_operation, trace_lines

    out = {}
    rng = np.random.default_rng(77)
    for i, (op, ext, kext, dt) in enumerate(DISPATCH_SPECS):
        R = len(ext)
        if op == "sdpa":
            S, d = sum(ext), 8
            q = rng.standard_normal((S, d)).astype(dt)
            k = rng.standard_normal((sum(kext), d)).astype(dt)
            v = rng.standard_normal((sum(kext), d)).astype(dt)
            ins = {"q": q, "k": k, "v": v}
        else:
            a = rng.standard_normal((sum(ext), 6)).astype(dt)
            b = rng.standard_normal((6, 5)).astype(dt)
            ins = {"a": a, "b": b}

        def prog(ctx, op=op, ins=ins, ext=ext, kext=kext):
            root = ctx.rank_id == 0
            if op == "sdpa":
                qs = scatter_global(ctx, ins["q"] if root else None, (Shard(0),), {0: ext})
                ks = scatter_global(ctx, ins["k"] if root else None, (Shard(0),), {0: kext})
                vs = scatter_global(ctx, ins["v"] if root else None, (Shard(0),), {0: kext})
                res = dispatch_operation("sdpa", qs, ks, vs)
            else:
                sa = scatter_global(ctx, ins["a"] if root else None, (Shard(0),), {0: ext})
                res = dispatch_operation("matmul", sa, replicated(ctx, ins["b"]))
            return (res.local, {int(a): list(e) for a, e in res.shard_shapes.items()},
                    [str(p) for p in res.placements], trace_lines(ctx)[-1])

        res = spawn_mesh((R,), ("domain",), prog)
        for n, arr in ins.items():
            out[f"f{i}_{n}"] = arr
        for r, (loc, shapes, pl, line) in enumerate(res):
            out[f"f{i}_local{r}"] = loc
        out[f"f{i}_meta"] = np.array(json.dumps({
            "op": op, "ext": list(ext), "kext": None if kext is None else list(kext),
            "shapes": res[0][1], "placements": res[0][2], "trace": res[0][3]}))
    out["count"] = np.array(len(DISPATCH_SPECS))
    return out


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None
    if only in (None, "core"):
        with open(os.path.join(HERE, "plans.json"), "w") as f:
            json.dump(make_plans(), f, indent=0)
        np.savez_compressed(os.path.join(HERE, "conv_cases.npz"), **make_conv_cases())
        np.savez_compressed(os.path.join(HERE, "ring_cases.npz"), **make_ring_cases())
        np.savez_compressed(os.path.join(HERE, "redist_cases.npz"), **make_redist_cases())
    if only in (None, "layers"):
        np.savez_compressed(os.path.join(HERE, "layer_cases.npz"), **make_layer_cases())
    if only in (None, "dispatch"):
        np.savez_compressed(os.path.join(HERE, "dispatch_cases.npz"), **make_dispatch_cases())
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
