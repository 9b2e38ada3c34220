"""The C-ABI communicator layer (csrc/comm.cu, comm.py) on one B200.

One GPU allows a one-rank NCCL world: self send/recv rounds (NCCL supports
them), one-rank all-reduces, splits, the watchdog and the error mapping,
and the NativeTransport mesh end to end (spawn_mesh backend "nccl", one
process).  Multi-rank NCCL needs distinct GPUs; its host logic (peer
lists, grouping, bytes) is the same code path.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(autouse=True)
def _need_gpu():
    from conftest import gpu_ready

    if not gpu_ready():
        pytest.fail("gpu tests need CUDA and libdpb200.so (no CPU path exists)")


def comm_mod():
    from paper_2605_11111_b200 import comm

    return comm


def world1():
    c = comm_mod()
    return c.NcclComm.init(1, 0, c.unique_id())


def test_nccl_loads_and_reports_version():
    assert comm_mod().version() >= 21800


def test_self_exchange_round_bytes_in_memory_order():
    w = world1()
    try:
        src = torch.randn((1, 16, 2, 12, 40), device=DEV).to(torch.bfloat16).contiguous(
            memory_format=torch.channels_last_3d)
        dst = torch.empty_like(src)
        flat_s = src.as_strided((src.numel(),), (1,))
        flat_d = dst.as_strided((dst.numel(),), (1,))
        w.exchange([(0, False, flat_s), (0, True, flat_d)])
        w.wait(timeout=30)
        assert torch.equal(dst, src)
        a = torch.arange(1000, device=DEV, dtype=torch.float32)
        b = torch.zeros_like(a)
        w.halo_sendrecv(-1, 0, None, a, None, b)
        w.wait(timeout=30)
        assert torch.equal(a, b)
        r = torch.zeros_like(a)
        w.ring_step(a, r)          # one rank: no-op
        w.wait(timeout=30)
        assert not r.any()
    finally:
        w.destroy()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_one_rank_allreduce_and_split(dtype):
    w = world1()
    try:
        x = torch.randn(777, device=DEV).to(dtype)
        for op in ("sum", "max"):
            out = torch.empty_like(x)
            w.allreduce(x, out, op)
            w.wait(torch.cuda.current_stream(), 30)
            assert torch.equal(out, x)
        s = w.split(color=0, key=0)
        assert (s.rank, s.size) == (0, 1)
        none = w.split(color=-1, key=0)
        assert none is None
        s.destroy()
    finally:
        w.destroy()


def test_comm_errors_map_to_package_errors():
    import paper_2605_11111_b200 as m

    w = world1()
    try:
        t = torch.zeros(8, device=DEV)
        with pytest.raises(m.DomainParError):
            w.exchange([(3, False, t)])          # peer outside the communicator
    finally:
        w.destroy()
    with pytest.raises(m.CollectiveError):
        comm_mod().NcclComm.init(1, 0, b"short")


def _native_prog(ctx):
    import paper_2605_11111_b200 as m

    assert type(ctx.transport).__name__ == "NativeTransport"
    x = torch.randn((1, 16, 6, 8, 40)).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last_3d)
    st = m.scatter_global(ctx, x, (m.Shard(2),))
    w = (torch.randn((32, 16, 3, 3, 3)) * 0.1).to(torch.bfloat16).to(ctx.device)
    y, tape = m.halo_conv_forward(st, w, 1, 1)
    dx, dw = m.halo_conv_backward(tape, torch.ones_like(y.local))
    g = m.all_reduce(ctx.axis_group(), dw, "sum")
    m.barrier(ctx.axis_group())
    want = m.dense_conv(x.to(ctx.device), w, 1, 1)
    return (y.local.float().cpu().numpy(), want.float().cpu().numpy(),
            torch.equal(g, dw))


def test_native_transport_one_rank_mesh():
    import paper_2605_11111_b200 as m

    (y, want, same), = m.spawn_mesh((1,), ("domain",), _native_prog, backend="nccl", timeout=120)
    assert same
    assert np.array_equal(y, want)
