"""The one-process-per-rank path (DistTransport — what bench.py / init_mesh
run with NCCL on N GPUs) driven end to end with the real sm_100a kernels: two
processes share the one GPU of the test box over gloo ("gloo-cuda" mesh,
device payloads staged through host memory, since NCCL refuses two ranks on
one device).  Halo conv fwd + bwd, ring attention fwd + bwd, redistribute and
a sharded layer norm against the fp64 oracle / exact slices."""

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import attention as oatt
from oracle import conv as oconv
from oracle import layers as olay

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


def _data():
    rng = np.random.default_rng(42)
    x = rng.standard_normal((1, 16, 16, 6, 40))
    w = rng.standard_normal((32, 16, 3, 3, 3)) * 0.1
    dy = rng.standard_normal((1, 32, 16, 6, 40))
    q, k, v, do = (rng.standard_normal((512, 2, 64)) for _ in range(4))
    g = rng.standard_normal((37, 23)).astype(np.float32)
    return x, w, dy, q, k, v, do, g


def _prog(ctx):
    import paper_2605_11111_b200 as dp

    x, w, dy, q, k, v, do, g = _data()
    dev = ctx.device
    r = ctx.rank_id
    cl = torch.channels_last_3d
    # halo conv fwd + bwd, D-sharded (9, 7), bf16 channels-last on the tcgen05 path
    ext = (9, 7)
    lo = sum(ext[:r])
    xl = torch.tensor(x[:, :, lo:lo + ext[r]]).to(torch.bfloat16).to(dev).contiguous(memory_format=cl)
    st = dp.ShardTensor(xl, x.shape, ctx, (dp.Shard(2),), {0: ext})
    wt = torch.tensor(w).to(torch.bfloat16).to(dev)
    before = ctx.collective_count
    y, tape = dp.halo_conv_forward(st, wt, 1, 1)
    oext = y.shard_shapes[0]
    olo = sum(oext[:r])
    dyl = torch.tensor(dy[:, :, olo:olo + oext[r]]).to(torch.bfloat16).to(dev).contiguous(memory_format=cl)
    dx, dw = dp.halo_conv_backward(tape, dyl)
    conv_colls = ctx.collective_count - before
    yfull, dxfull = y.full_tensor(), dx.full_tensor()
    # ring attention fwd + bwd over uneven (200, 312) query / key shards
    qe, ke = (200, 312), (312, 200)
    qlo, klo = sum(qe[:r]), sum(ke[:r])
    mk = lambda a, e, l0: dp.ShardTensor(  # noqa: E731
        torch.tensor(a[l0:l0 + e[r]]).to(torch.bfloat16).to(dev), a.shape, ctx, (dp.Shard(0),),
        {0: e})
    qs, ks, vs = mk(q, qe, qlo), mk(k, ke, klo), mk(v, ke, klo)
    before = ctx.collective_count
    o, atape = dp.ring_attention_forward(qs, ks, vs)
    ring_colls = ctx.collective_count - before
    dq, dk, dv = dp.ring_attention_backward(
        atape, torch.tensor(do[qlo:qlo + qe[r]]).to(torch.bfloat16).to(dev))
    ofull, dqf, dkf, dvf = (t.full_tensor() for t in (o, dq, dk, dv))
    # redistribute Shard(0) (uneven) -> Shard(1) and the round trip back
    ge = (30, 7)
    gl = torch.tensor(g[sum(ge[:r]):sum(ge[:r]) + ge[r]]).to(dev)
    gs = dp.ShardTensor(gl, g.shape, ctx, (dp.Shard(0),), {0: ge})
    s1 = dp.redistribute(gs, (dp.Shard(1),))
    back = dp.redistribute(s1, (dp.Shard(0),))
    # sharded layer norm over the sharded dim (one all_reduce)
    ln = dp.dispatch_operation("layer_norm", gs, 0)
    return (yfull, dxfull, dw, conv_colls, ofull, dqf, dkf, dvf, ring_colls, s1.local,
            s1.shard_shapes, back.full_tensor(), ln.full_tensor())


def test_process_mesh_end_to_end_on_one_gpu():
    import paper_2605_11111_b200 as dp

    res = dp.spawn_mesh((2,), ("domain",), _prog, backend="gloo-cuda", timeout=120)
    x, w, dy, q, k, v, do, g = _data()
    bf = lambda a: torch.tensor(a).to(torch.bfloat16).double().numpy()  # noqa: E731
    xr, wr, dyr = bf(x), bf(w), bf(dy)
    want_y = oconv.conv(xr, wr, 1, 1)
    want_dx, want_dw = oconv.conv_grads(xr, wr, dyr, 1, 1)
    qr, kr, vr, dor = bf(q), bf(k), bf(v), bf(do)
    want_o = oatt.sdpa(qr, kr, vr)
    want_dq, want_dk, want_dv = oatt.sdpa_grads(qr, kr, vr, dor)
    for r, out in enumerate(res):
        (yfull, dxfull, dw, conv_colls, ofull, dqf, dkf, dvf, ring_colls, s1, s1_shapes, back,
         ln) = out
        f = lambda t: t.float().numpy().astype(np.float64)  # noqa: E731
        assert rel_err(f(yfull), want_y) < 1e-2
        assert rel_err(f(dxfull), want_dx) < 1e-2
        assert rel_err(f(dw), want_dw) < 2e-2
        assert conv_colls == 3          # halo + reverse halo + dW all-reduce
        assert rel_err(f(ofull), want_o) < 1.5e-2
        assert rel_err(f(dqf), want_dq) < 2e-2
        assert rel_err(f(dkf), want_dk) < 2e-2
        assert rel_err(f(dvf), want_dv) < 2e-2
        assert ring_colls == 1          # R - 1 K||V hops
        c = dp.default_chunk(23, 2)
        assert torch.equal(s1, torch.tensor(g[:, sum(c[:r]):sum(c[:r]) + c[r]]))
        assert s1_shapes == {0: tuple(c)}
        assert torch.equal(back, torch.tensor(g))
        assert rel_err(ln.numpy(), olay.layer_norm(g, 0)) < 1e-5


def _autograd_prog(ctx):
    """halo_conv_autograd (replicated ShardTensor weight) and
    ring_attention_autograd through torch.autograd on the process mesh."""
    import paper_2605_11111_b200 as dp

    x, w, dy, q, k, v, do, _ = _data()
    dev = ctx.device
    r = ctx.rank_id
    cl = torch.channels_last_3d
    ext = (9, 7)
    lo = sum(ext[:r])
    xl = torch.tensor(x[:, :, lo:lo + ext[r]]).to(torch.bfloat16).to(dev) \
        .contiguous(memory_format=cl).requires_grad_(True)
    st = dp.ShardTensor(xl, x.shape, ctx, (dp.Shard(2),), {0: ext})
    wl = torch.tensor(w).to(torch.bfloat16).to(dev).requires_grad_(True)
    wst = dp.ShardTensor(wl, w.shape, ctx, (dp.Replicate(),), {})
    y = dp.halo_conv_autograd(st, wst, 1, 1)
    oext = y.shard_shapes[0]
    olo = sum(oext[:r])
    dyl = torch.tensor(dy[:, :, olo:olo + oext[r]]).to(torch.bfloat16).to(dev) \
        .contiguous(memory_format=cl)
    y.local.backward(dyl)
    dx = dp.ShardTensor(xl.grad, x.shape, ctx, (dp.Shard(2),), {0: ext}).full_tensor()
    qe = (256, 256)
    mk = lambda a: torch.tensor(a[r * 256:(r + 1) * 256]).to(torch.bfloat16).to(dev) \
        .requires_grad_(True)  # noqa: E731
    ql, kl, vl = mk(q), mk(k), mk(v)
    qs, ks, vs = (dp.ShardTensor(t, q.shape, ctx, (dp.Shard(0),), {0: qe}) for t in (ql, kl, vl))
    o = dp.ring_attention_autograd(qs, ks, vs)
    o.local.backward(torch.tensor(do[r * 256:(r + 1) * 256]).to(torch.bfloat16).to(dev))
    grads = [dp.ShardTensor(t.grad, q.shape, ctx, (dp.Shard(0),), {0: qe}).full_tensor()
             for t in (ql, kl, vl)]
    return (y.full_tensor(), dx, wl.grad.float().cpu(), o.full_tensor(), *grads)


def test_autograd_wrappers_on_process_mesh():
    import paper_2605_11111_b200 as dp

    res = dp.spawn_mesh((2,), ("domain",), _autograd_prog, backend="gloo-cuda", timeout=120)
    x, w, dy, q, k, v, do, _ = _data()
    bf = lambda a: torch.tensor(a).to(torch.bfloat16).double().numpy()  # noqa: E731
    xr, wr, dyr = bf(x), bf(w), bf(dy)
    want_y = oconv.conv(xr, wr, 1, 1)
    want_dx, want_dw = oconv.conv_grads(xr, wr, dyr, 1, 1)
    qr, kr, vr, dor = bf(q), bf(k), bf(v), bf(do)
    want = [oatt.sdpa(qr, kr, vr), *oatt.sdpa_grads(qr, kr, vr, dor)]
    f = lambda t: t.float().numpy().astype(np.float64)  # noqa: E731
    for y, dx, dw, o, dq, dk, dv in res:
        assert rel_err(f(y), want_y) < 1e-2
        assert rel_err(f(dx), want_dx) < 1e-2
        assert rel_err(f(dw), want_dw) < 3e-2          # bf16 weight gradient (cast back)
        assert rel_err(f(o), want[0]) < 1.5e-2
        for got, exp in zip((dq, dk, dv), want[1:]):
            assert rel_err(f(got), exp) < 2e-2


def test_autograd_wrappers_refuse_thread_mesh():
    import paper_2605_11111_b200 as dp

    def prog(ctx):
        xl = torch.zeros((1, 16, 4, 8, 16), dtype=torch.bfloat16, device=ctx.device)
        st = dp.ShardTensor(xl, (1, 16, 4, 8, 16), ctx, (dp.Shard(2),), {0: (4,)})
        with pytest.raises(dp.UnsupportedConfigError, match="one process per rank"):
            dp.halo_conv_autograd(st, torch.zeros((16, 16, 3, 3, 3), dtype=torch.bfloat16,
                                                  device=ctx.device), 1, 1)
        q = dp.ShardTensor(torch.zeros((8, 64), dtype=torch.bfloat16, device=ctx.device),
                           (8, 64), ctx, (dp.Shard(0),), {0: (8,)})
        with pytest.raises(dp.UnsupportedConfigError, match="one process per rank"):
            dp.ring_attention_autograd(q, q, q)
        return True

    assert dp.spawn_mesh((1,), ("domain",), prog)[0]
