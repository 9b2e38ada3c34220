"""Device kernels vs the oracle: strided copy / accumulate, conv fwd/dgrad/
wgrad over the virtual halo block, attention block fold (SIMT and tcgen05)."""

import math

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


def kernels():
    from paper_2605_11111_b200 import kernels as k

    return k


@pytest.mark.parametrize("shape,perm,sl", [
    ((64, 33, 7), (0, 1, 2), (slice(None), slice(3, 20), slice(None))),
    ((8, 16, 128), (2, 0, 1), (slice(None), slice(None), slice(5, 70))),
    ((1, 32, 9, 256, 256), (0, 1, 2, 3, 4), (slice(None), slice(None), slice(0, 2))),
    ((4, 4096), (0, 1), (slice(None), slice(1000, 3000))),
    ((3, 5, 7, 11), (3, 1, 0, 2), (slice(1, 3),)),
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64, torch.int64])
def test_copy_strided_matches_slicing(shape, perm, sl, dtype):
    src = torch.randn(shape, device=DEV).to(dtype) if dtype.is_floating_point else \
        torch.randint(-1000, 1000, shape, device=DEV, dtype=dtype)
    view = src.permute(perm)[sl] if len(sl) <= len(shape) else src.permute(perm)
    out = torch.empty(view.shape, dtype=dtype, device=DEV)
    kernels().copy_strided(out, view)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), view.cpu())  # bit-exact


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_accumulate_strided(dtype):
    base = torch.randn(4, 6, 10, device=DEV).to(dtype)
    add = torch.randn(4, 2, 10, device=DEV).to(dtype)
    want = base.clone().float()
    want[:, 1:3] += add.float()
    kernels().accumulate(base[:, 1:3], add)
    got = base.float()
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-6
    assert torch.allclose(got.cpu(), want.to(dtype).float().cpu(), atol=tol, rtol=tol)


def _conv_case(rng, nsp, batch, cin, cout, sp, k, s, p, dtype):
    x = rng.standard_normal((batch, cin) + sp)
    w = rng.standard_normal((cout, cin) + (k,) * nsp) * 0.3
    return x, w


CONV_CASES = [
    # nsp, batch, cin, cout, spatial, k, stride, pad
    (1, 2, 3, 4, (17,), 3, 1, 1),
    (1, 1, 2, 3, (20,), 5, 2, 3),
    (2, 2, 3, 5, (12, 9), 3, 1, 1),
    (2, 1, 4, 2, (11, 13), 5, 2, 2),
    (2, 1, 16, 32, (24, 40), 3, 1, 1),
    (3, 1, 4, 6, (7, 8, 9), 3, 1, 1),
    (3, 1, 16, 32, (6, 10, 20), 3, 1, 1),
    (3, 2, 3, 2, (7, 6, 9), 3, 2, 0),
]


def _layouts(x, channels_last):
    if not channels_last or x.dim() < 4:
        return x
    fmt = torch.channels_last if x.dim() == 4 else torch.channels_last_3d
    return x.contiguous(memory_format=fmt)


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("algo", ["simt", "auto"])
def test_dense_conv_fwd_bwd_vs_oracle(case, dtype, algo):
    """Unsharded conv: fwd, dgrad, wgrad against the fp64 oracle."""
    from paper_2605_11111_b200 import ops

    k = kernels()
    prev = k.set_algo(algo)
    try:
        nsp, batch, cin, cout, sp, ks, s, p = case
        rng = np.random.default_rng(hash(case) % 2**32)
        x, w = _conv_case(rng, nsp, batch, cin, cout, sp, ks, s, p, dtype)
        xt = _layouts(torch.tensor(x, device=DEV).to(dtype), algo == "auto")
        wt = torch.tensor(w, device=DEV).to(dtype)
        y = ops.dense_conv(xt, wt, s, p)
        # oracle on the (rounded) inputs, fp64
        xr, wr = to_np(xt).astype(np.float64), to_np(wt).astype(np.float64)
        want = oconv.conv(xr, wr, s, p)
        tol = {torch.float64: 1e-12, torch.float32: 1e-5, torch.bfloat16: 1e-2}[dtype]
        assert rel_err(to_np(y), want) < tol
        dy = rng.standard_normal(want.shape)
        dyt = _layouts(torch.tensor(dy, device=DEV).to(dtype), algo == "auto")
        from paper_2605_11111_b200.sharding import ShardTensor
        from paper_2605_11111_b200 import spawn_mesh, replicated

        def prog(ctx):
            xs = replicated(ctx, xt)
            out, tape = ops.halo_conv_forward(xs, wt, s, p)
            dx, dw = ops.halo_conv_backward(tape, dyt)
            return dx.local, dw

        dx, dw = spawn_mesh((1,), ("domain",), prog)[0]
        dxr, dwr = oconv.conv_grads(xr, wr, to_np(dyt).astype(np.float64), s, p)
        assert rel_err(to_np(dx), dxr) < tol
        assert rel_err(to_np(dw), dwr) < (tol if dtype != torch.bfloat16 else 2e-2)
    finally:
        k.set_algo(prev)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("sq,sk,h,d", [(5, 11, 1, 6), (37, 50, 3, 16), (130, 260, 2, 64),
                                        (64, 128, 4, 128), (1, 1, 1, 4)])
def test_attention_block_fold_vs_oracle(dtype, sq, sk, h, d):
    """Fold K/V in 3 uneven blocks through the state kernel == dense sdpa."""
    from paper_2605_11111_b200 import ops

    rng = np.random.default_rng(sq * 7 + sk)
    q = torch.tensor(rng.standard_normal((sq, h, d)), device=DEV).to(dtype)
    k_ = torch.tensor(rng.standard_normal((sk, h, d)), device=DEV).to(dtype)
    v = torch.tensor(rng.standard_normal((sk, h, d)), device=DEV).to(dtype)
    cuts = [0, sk // 3, sk // 3, sk]  # includes an empty block
    blocks = [(k_[a:b], v[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    out, lse = ops._attn_local(q, blocks, 1.0 / math.sqrt(d))
    want = oatt.sdpa(to_np(q).astype(np.float64), to_np(k_).astype(np.float64),
                     to_np(v).astype(np.float64))
    tol = {torch.float64: 1e-12, torch.float32: 1e-5, torch.bfloat16: 1.5e-2}[dtype]
    assert rel_err(to_np(out), want) < tol
