"""Oracle parity at BASELINE.json's full sizes.

* cfg1 (the reference's own CPU parity anchor): conv2d 3x3 on the full
  1x32x1024x1024 fp32 grid, H-sharded over R = 2, forward + backward against
  the oracle (the reference's dense.conv einsum, bitwise-pinned; fp64
  adjoint) at the reference's fp32 tolerance 1e-5.
* cfg2 at R = 8: the 1x16x256^3 bf16 UNet block conv(16->32) -> conv(32->32)
  forward + input gradient, checked on boxes straddling EVERY shard boundary
  (and the volume's corners) against oracle.stack_window, at 1e-2.
* cfg3 at R = 8: 64k tokens x 16 heads x 64, bf16 ring attention forward +
  backward; for two heads a 128-query-row slab (o, dq, every key) and a
  128-key slab (dk, dv, every query) against oracle.head_slab, and for all
  heads the exact identity sum_j dV_j = sum_i dO_i.
"""

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


def test_cfg1_full_grid_fwd_bwd_vs_oracle():
    import paper_2605_11111_b200 as m

    rng = np.random.default_rng(101)
    G, C = 1024, 32
    x = rng.standard_normal((1, C, G, G)).astype(np.float32)
    w = (rng.standard_normal((C, C, 3, 3)) * 0.1).astype(np.float32)
    dy = rng.standard_normal((1, C, G, G)).astype(np.float32)
    want_y = oconv.conv(x, w, 1, 1)                    # the reference's fp32 einsum
    want_dx, want_dw = oconv.conv_grads(x, w, dy, 1, 1)
    xt, wt, dyt = torch.tensor(x), torch.tensor(w), torch.tensor(dy)
    ext = m.default_chunk(G, 2)

    def prog(ctx):
        st = m.scatter_global(ctx, xt if ctx.rank_id == 0 else None, (m.Shard(2),))
        out, tape = m.halo_conv_forward(st, wt.to(DEV), 1, 1)
        lo, hi = out.shard_interval(0)
        dx, dw = m.halo_conv_backward(tape, dyt[:, :, lo:hi].to(DEV))
        return out.local.cpu(), dx.local.cpu(), dw.cpu(), out.shard_shapes[0]

    res = m.spawn_mesh((2,), ("domain",), prog)
    assert tuple(res[0][3]) == (513, 511)               # the reference's anchor ownership
    y = torch.cat([r[0] for r in res], dim=2)
    dx = torch.cat([r[1] for r in res], dim=2)
    assert rel_err(to_np(y), want_y) < 1e-5
    assert rel_err(to_np(dx), want_dx) < 1e-5
    for r in res:
        assert rel_err(to_np(r[2]), want_dw) < 1e-5
    assert [int(e) for e in ext] == [512, 512]


def _boxes(G, bounds, d_half=3):
    """D boxes around every boundary (and both volume ends) x two H/W boxes
    (a corner box touching the zero padding, an interior box)."""
    out = []
    for b in [0] + list(bounds) + [G]:
        lo_d, hi_d = max(0, b - d_half), min(G, b + d_half)
        for (h0, w0) in ((0, 0), (G // 2 - 4, G - 16)):
            out.append(((lo_d, h0, w0), (hi_d, h0 + 8, w0 + 16)))
    return out


def test_cfg2_r8_boundary_slabs_vs_oracle():
    import paper_2605_11111_b200 as m

    G, C0, C1, R = 256, 16, 32, 8
    gen = torch.Generator().manual_seed(202)
    x = torch.randn((1, C0, G, G, G), generator=gen).to(torch.bfloat16)
    w1 = (torch.randn((C1, C0, 3, 3, 3), generator=gen) * 0.05).to(torch.bfloat16)
    w2 = (torch.randn((C1, C1, 3, 3, 3), generator=gen) * 0.05).to(torch.bfloat16)
    g = torch.randn((1, C1, G, G, G), generator=gen).to(torch.bfloat16)
    cl = torch.channels_last_3d
    x_cl, g_cl = x.contiguous(memory_format=cl), g.contiguous(memory_format=cl)

    def prog(ctx):
        st = m.scatter_global(ctx, x_cl if ctx.rank_id == 0 else None, (m.Shard(2),))
        y1, t1 = m.halo_conv_forward(st, w1.to(DEV), 1, 1)
        y2, t2 = m.halo_conv_forward(y1, w2.to(DEV), 1, 1)
        lo, hi = y2.shard_interval(0)
        dy1, _ = m.halo_conv_backward(t2, g_cl[:, :, lo:hi].to(DEV))
        dx, _ = m.halo_conv_backward(t1, dy1)
        return y2.local.cpu(), dx.local.cpu(), list(y2.shard_shapes[0])

    from paper_2605_11111_b200 import kernels

    simt0 = kernels.simt_count()
    res = m.spawn_mesh((R,), ("domain",), prog, device=DEV)
    assert kernels.simt_count() == simt0
    y2 = torch.cat([r[0] for r in res], dim=2)
    dx = torch.cat([r[1] for r in res], dim=2)
    assert res[0][2] == [34] + [32] * 6 + [30]          # drift of two same-pad layers
    ws = [to_np(w1).astype(np.float64), to_np(w2).astype(np.float64)]
    ws_t = [oconv.transposed_flipped(ws[1]), oconv.transposed_flipped(ws[0])]
    bounds = [32 * r for r in range(1, R)]
    out_bounds = list(np.cumsum(res[0][2])[:-1])
    for lo, hi in _boxes(G, sorted(set(bounds) | set(int(b) for b in out_bounds))):
        want = oconv.stack_window(x, ws, lo, hi)
        got = to_np(y2[:, :, lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]])
        assert rel_err(got, want) < 1e-2, (lo, hi)
        want = oconv.stack_window(g, ws_t, lo, hi)
        got = to_np(dx[:, :, lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]])
        assert rel_err(got, want) < 1e-2, (lo, hi)


def test_cfg3_r8_slabs_and_identities_vs_oracle():
    import paper_2605_11111_b200 as m

    S, H, D, R = 65536, 16, 64, 8
    gen = torch.Generator().manual_seed(303)
    q, k, v, do = (torch.randn((S, H, D), generator=gen).to(torch.bfloat16) for _ in range(4))
    ext = m.default_chunk(S, R)

    def prog(ctx):
        root = ctx.rank_id == 0
        qs, ks, vs = (m.scatter_global(ctx, t if root else None, (m.Shard(0),))
                      for t in (q, k, v))
        out, tape = m.ring_attention_forward(qs, ks, vs)
        lo, hi = out.shard_interval(0)
        dq, dk, dv = m.ring_attention_backward(tape, do[lo:hi].to(DEV))
        return [t.cpu() for t in (out.local, dq.local, dk.local, dv.local)]

    res = m.spawn_mesh((R,), ("domain",), prog, device=DEV)
    o, dq, dk, dv = (torch.cat([r[i] for r in res], dim=0) for i in range(4))
    qn, kn, vn, don = (to_np(t) for t in (q, k, v, do))
    # slabs straddling a shard boundary, in two heads
    rows = slice(ext[0] - 64, ext[0] + 64)
    keys = slice(3 * ext[0] - 64, 3 * ext[0] + 64)
    for h in (0, 11):
        so, sdq, sdk, sdv = oatt.head_slab(qn[:, h], kn[:, h], vn[:, h], don[:, h], rows, keys)
        assert rel_err(to_np(o[rows, h]), so) < 1.5e-2
        assert rel_err(to_np(dq[rows, h]), sdq, 1.0) < 2e-2
        assert rel_err(to_np(dk[keys, h]), sdk, 1.0) < 2e-2
        assert rel_err(to_np(dv[keys, h]), sdv, 1.0) < 2e-2
    # exact identity at full length, every head and channel: sum_j dV_j =
    # sum_i dO_i (every softmax row sums to one)
    sdv_all = dv.double().sum(dim=0)
    sdo_all = do.double().sum(dim=0)
    assert float((sdv_all - sdo_all).abs().max()) < 1e-2 * float(sdo_all.abs().max())
