"""The sharded conv hot path stays on the tensor cores.

cfg2-shaped UNet encoder block conv(16->32) -> conv(32->32), 3x3x3, s1 p1,
W = 256, channels-last bf16, D-sharded over R = 4 and R = 8 thread-ranks
(even and uneven extents), forward + backward through the public
`halo_conv_forward` / `halo_conv_backward`, checked against the fp64 oracle
(oracle/conv.py).  Every conv launch — interior rows, halo rows, the dgrad
with its reverse-halo output, the wgrad over the received halo — must run on
the tcgen05 kernels: the library's algorithm is forced to "strict" (an
UnsupportedConfigError instead of any CUDA-core detour), the library's
CUDA-core call counter must not move, and the CUDA kernel names captured by
the profiler must contain no CUDA-core conv kernel.
"""

import numpy as np
import pytest
import torch

from conftest import rel_err, to_np
from oracle import conv as oconv

pytestmark = pytest.mark.gpu
DEV = "cuda"
CL = torch.channels_last_3d
SIMT_KERNELS = ("conv_fwd_simt", "conv_dgrad_simt", "conv_wgrad_partial", "wgrad_reduce",
                "conv_tiled")


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


def cuda_kernels(fn):
    """Run fn() under the CUDA profiler; return (result, kernel names)."""
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    return res, names


BLOCK_CASES = [
    (4, (4, 4, 4, 4), 8),
    (8, (4,) * 8, 8),
    (4, (6, 3, 5, 2), 6),
    (8, (3, 5, 2, 4, 4, 6, 3, 5), 4),
]


@pytest.mark.parametrize("R,ext,H", BLOCK_CASES)
def test_sharded_conv_block_on_tcgen05(R, ext, H):
    import paper_2605_11111_b200 as m
    from paper_2605_11111_b200 import kernels

    W, C0, C1 = 256, 16, 32
    D = sum(ext)
    rng = np.random.default_rng(R * 100 + D + H)
    x = torch.tensor(rng.standard_normal((1, C0, D, H, W))).to(torch.bfloat16)
    w1 = torch.tensor(rng.standard_normal((C1, C0, 3, 3, 3)) * 0.05).to(torch.bfloat16)
    w2 = torch.tensor(rng.standard_normal((C1, C1, 3, 3, 3)) * 0.05).to(torch.bfloat16)
    xr, w1r, w2r = (to_np(t).astype(np.float64) for t in (x, w1, w2))
    y1r = oconv.conv_fast(xr, w1r, 1, 1)
    y2r = oconv.conv_fast(y1r, w2r, 1, 1)
    g = torch.tensor(rng.standard_normal(y2r.shape)).to(torch.bfloat16)
    dy1r, dw2r = oconv.conv_grads(y1r, w2r, to_np(g).astype(np.float64), 1, 1)
    dxr, dw1r = oconv.conv_grads(xr, w1r, dy1r, 1, 1)

    def prog(ctx):
        st = m.scatter_global(ctx, x if ctx.rank_id == 0 else None, (m.Shard(2),), {0: ext})
        st = m.ShardTensor(st.local.contiguous(memory_format=CL), st.global_shape, ctx,
                           st.placements, st.shard_shapes)
        y1, t1 = m.halo_conv_forward(st, w1.to(DEV), 1, 1)
        y2, t2 = m.halo_conv_forward(y1, w2.to(DEV), 1, 1)
        assert y1.local.is_contiguous(memory_format=CL)
        if t1.halo is not None:
            assert t1.halo.is_contiguous(memory_format=CL)
        lo, hi = y2.shard_interval(0)
        gl = g[:, :, lo:hi].to(DEV).contiguous(memory_format=CL)
        dy1, dw2 = m.halo_conv_backward(t2, gl)
        dx, dw1 = m.halo_conv_backward(t1, dy1)
        return y2.full_tensor(), dx.full_tensor(), dw1, dw2

    prev = kernels.set_algo("strict")
    try:
        simt0 = kernels.simt_count()
        res, names = cuda_kernels(lambda: m.spawn_mesh((R,), ("domain",), prog, device=DEV))
        assert kernels.simt_count() == simt0, "a conv call left the tensor cores"
    finally:
        kernels.set_algo(prev)
    bad = sorted({n for n in names if any(s in n for s in SIMT_KERNELS)})
    assert not bad, f"CUDA-core conv kernels launched: {bad}"
    assert any("conv_tc_kernel" in n for n in names)
    assert any("conv_wgrad" in n for n in names)
    for y2, dx, dw1, dw2 in res:
        assert rel_err(to_np(y2), y2r) < 1e-2
        assert rel_err(to_np(dx), dxr) < 1e-2
        assert rel_err(to_np(dw1), dw1r) < 2e-2
        assert rel_err(to_np(dw2), dw2r) < 2e-2


def test_auto_counts_out_of_envelope_calls():
    """AUTO still serves shapes outside the tcgen05 envelope (here stride 2,
    as in the reference's own test-suite), but every such call is counted;
    STRICT refuses it with UnsupportedConfigError."""
    import paper_2605_11111_b200 as m
    from paper_2605_11111_b200 import kernels

    x = torch.randn((1, 16, 9, 40), device=DEV).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    w = torch.randn((16, 16, 3, 3), device=DEV).to(torch.bfloat16)
    c0 = kernels.simt_count()
    m.dense_conv(x, w, stride=2, padding=1)
    assert kernels.simt_count() == c0 + 1
    c1 = kernels.simt_count()
    m.dense_conv(x, w, stride=1, padding=1)
    assert kernels.simt_count() == c1
    prev = kernels.set_algo("strict")
    try:
        with pytest.raises(m.UnsupportedConfigError):
            m.dense_conv(x, w, stride=2, padding=1)
    finally:
        kernels.set_algo(prev)
