"""CPU workloads of the benchmark's baseline legs (TEST INFRASTRUCTURE):
the bench step restated with the oracle, for bounded samples of the
configured workload.  Used only by bench.py's `cpu_baseline` and
`--impl reference` legs."""

import numpy as np

from . import attention, conv


def conv_block_step(x, w1, w2, g, pad=1):
    """fwd+bwd of the UNet-style block conv(w1) -> conv(w2) on an fp32
    sub-volume with upstream gradient g of the block output (the reference
    computes in fp32; its conv is dense.conv's einsum, restated in conv.py;
    the backward, which the reference lacks, runs in fp32 too).
    Returns (dx, dw1, dw2)."""
    y1 = conv.conv(x, w1, 1, pad)
    y2 = conv.conv(y1, w2, 1, pad)
    assert y2.shape == g.shape
    dy1, dw2 = conv.conv_grads(y1, w2, g, 1, pad, np.float32)
    dx, dw1 = conv.conv_grads(x, w1, dy1, 1, pad, np.float32)
    return dx, dw1, dw2


def conv_stack_step(x, ws, g, pad=1):
    """fwd+bwd of an L-layer 2-D conv stack (cfg4) on an fp32 sample."""
    acts = [x]
    for w in ws:
        acts.append(conv.conv(acts[-1], w, 1, pad))
    dy = g
    dws = []
    for w, a in zip(reversed(ws), reversed(acts[:-1])):
        dy, dw = conv.conv_grads(a, w, dy, 1, pad, np.float32)
        dws.append(dw)
    return dy, dws[::-1]


def attention_step(q, k, v, do):
    """fwd+bwd of single-rank attention on an fp32 sample (fp64 softmax)."""
    out = attention.sdpa(q, k, v)
    return out, attention.sdpa_grads(q, k, v, do)
