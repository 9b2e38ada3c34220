"""Convolution restated from the reference (TEST INFRASTRUCTURE).

conv()       domainpar/dense.py:174-214 — np.pad + sliding_window_view +
             einsum, with the reference's einsum specs for 1-D/2-D; the 3-D
             spec 'bcpqrklm,dcklm->bdpqr' extends the same construction (the
             reference rejects 3-D, dense.py:181-185).
conv_fast()  the same convolution summed tap by tap with BLAS matmuls in
             float64 (large parity cases), pinned against conv().
conv_grads() the adjoint: dX by scattering dY*W back over every window
             position, dW by contracting the windows with dY.  No reference
             function exists (no autograd); pinned by central
             finite differences in tests/test_oracle.py.
stack_window() a box of the output of a stack of stride-1 same-padded convs
             computed from the input box it depends on (zero padding only at
             the global borders): full-size parity on slabs.
halo_conv_members()  per-member outputs of the sharded algorithm
             (domainpar/ops.py:363-422) on the gathered input.
"""

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

from .plan import conv_out, member_plans

_SPECS = {1: "bcok,dck->bdo", 2: "bcpqkl,dckl->bdpq", 3: "bcpqrklm,dcklm->bdpqr"}


def _norm(n, v):
    return (v,) * n if isinstance(v, int) else tuple(v)


def conv(x, w, stride=1, padding=0):
    n = w.ndim - 2
    batched = x.ndim == n + 2
    xb = x if batched else x[None]
    strides, pads = _norm(n, stride), _norm(n, padding)
    for g, k, s, p in zip(xb.shape[2:], w.shape[2:], strides, pads):
        conv_out(g, k, s, p)
    xp = np.pad(xb, [(0, 0), (0, 0)] + [(p, p) for p in pads])
    win = sliding_window_view(xp, w.shape[2:], axis=tuple(range(2, 2 + n)))
    win = win[(slice(None), slice(None)) + tuple(slice(None, None, s) for s in strides)]
    out = np.ascontiguousarray(np.einsum(_SPECS[n], win, w), dtype=x.dtype)
    return out if batched else out[0]


def conv_fast(x, w, stride=1, padding=0):
    """conv() with the same zero padding and window arithmetic, summed tap by
    tap as BLAS matmuls in float64 (Y += W_tap X_tap) instead of the
    reference's single einsum: the oracle for the large parity cases, pinned
    against conv() in tests/test_oracle.py.  Returns float64."""
    n = w.ndim - 2
    batched = x.ndim == n + 2
    xb = (x if batched else x[None]).astype(np.float64)
    w64 = w.astype(np.float64)
    strides, pads = _norm(n, stride), _norm(n, padding)
    outs = [conv_out(g, k, s, p) for g, k, s, p in zip(xb.shape[2:], w.shape[2:], strides, pads)]
    xp = np.pad(xb, [(0, 0), (0, 0)] + [(p, p) for p in pads])
    nb, no = xb.shape[0], w.shape[0]
    y = np.zeros((nb, no, int(np.prod(outs))), dtype=np.float64)
    for tap in np.ndindex(*w.shape[2:]):
        sl = (slice(None), slice(None)) + tuple(
            slice(t, t + s * (o - 1) + 1, s) for t, s, o in zip(tap, strides, outs))
        xs = np.ascontiguousarray(xp[sl]).reshape(nb, xb.shape[1], -1)
        y += np.matmul(w64[(slice(None), slice(None)) + tap][None], xs)
    y = y.reshape((nb, no) + tuple(outs))
    return y if batched else y[0]


def conv_grads(x, w, dy, stride=1, padding=0, dtype=np.float64):
    """(dx, dw) of y = conv(x, w) given dy, computed in `dtype` (float64 for
    parity; the CPU baseline legs use float32, the reference's compute type)."""
    n = w.ndim - 2
    batched = x.ndim == n + 2
    xb = (x if batched else x[None]).astype(dtype)
    dyb = (dy if batched else dy[None]).astype(dtype)
    w64 = w.astype(dtype)
    strides, pads = _norm(n, stride), _norm(n, padding)
    xp = np.pad(xb, [(0, 0), (0, 0)] + [(p, p) for p in pads])
    dxp = np.zeros_like(xp)
    dw = np.zeros_like(w64)
    outs = dyb.shape[2:]
    for tap in np.ndindex(*w.shape[2:]):
        sl = (slice(None), slice(None)) + tuple(
            slice(t, t + s * (o - 1) + 1, s) for t, s, o in zip(tap, strides, outs))
        xs = xp[sl]                                     # [b, ci, *out]
        wt = w64[(slice(None), slice(None)) + tap]      # [co, ci]
        nb, no = dyb.shape[:2]
        dyf = dyb.reshape(nb, no, -1)
        # per-tap contractions as BLAS matmuls: dX_tap = W_tap^T dY, dW_tap = sum_b dY X_tap^T
        dxp[sl] += np.matmul(wt.T[None], dyf).reshape(xs.shape)
        xf = np.ascontiguousarray(xs).reshape(nb, xs.shape[1], -1)
        dw[(slice(None), slice(None)) + tap] = np.matmul(dyf, xf.transpose(0, 2, 1)).sum(0)
    crop = (slice(None), slice(None)) + tuple(slice(p, p + g) for p, g in zip(pads, xb.shape[2:]))
    dx = dxp[crop]
    return (dx if batched else dx[0]), dw


def halo_conv_members(x, w, extents, shard_dim, stride=1, padding=0):
    """Per-member local outputs of the sharded conv (ops.py:363-422) computed
    the reference's way: extended block = local + right-halo rows, trimmed
    to [max(w_min,0), min(w_max,G)), zero-padded, dense conv with the
    sharded padding materialised.  Returns (outputs, out_extents)."""
    n = w.ndim - 2
    first = x.ndim - n
    sp = shard_dim - first
    strides, pads = _norm(n, stride), _norm(n, padding)
    g_in = x.shape[shard_dim]
    k, s, p = w.shape[2 + sp], strides[sp], pads[sp]
    plans = member_plans(extents, g_in, k, s, p)
    bounds = np.concatenate([[0], np.cumsum(extents)]).astype(int)
    outs = []
    for m, (j_lo, j_hi, w_min, w_max, lw, rw) in enumerate(plans):
        a, b = bounds[m], bounds[m + 1]
        if j_hi == j_lo:
            shape = list(x.shape)
            shape[shard_dim] = 0
            shape[first - 1] = w.shape[0]
            for i in range(n):
                if i != sp:
                    shape[first + i] = conv_out(x.shape[first + i], w.shape[2 + i], strides[i],
                                                pads[i])
            outs.append(np.zeros(shape, dtype=x.dtype))
            continue
        lo, hi = max(w_min, 0), min(w_max, g_in)
        idx = [slice(None)] * x.ndim
        idx[shard_dim] = slice(lo, hi)
        block = x[tuple(idx)]
        pad = [(0, 0)] * x.ndim
        pad[shard_dim] = (max(0, -w_min), max(0, w_max - g_in))
        block = np.pad(block, pad)
        lp = list(pads)
        lp[sp] = 0
        outs.append(conv(block, w, strides, tuple(lp)))
    return outs, [pl[1] - pl[0] for pl in plans]


def transposed_flipped(w):
    """Weights of the input-gradient convolution of a stride-1 conv:
    wt[ci, co, t] = w[co, ci, k - 1 - t] (dX = conv(dY, wt, padding k-1-p))."""
    n = w.ndim - 2
    return np.ascontiguousarray(np.flip(w, axis=tuple(range(2, 2 + n))).swapaxes(0, 1))


def stack_window(x, ws, lo, hi):
    """Box [lo, hi) (per spatial dim) of the output of conv(...conv(x, ws[0])
    ..., ws[-1]), every layer stride 1 with padding (k-1)/2, computed from
    the input box it depends on: the global input is read (as float64) only
    there, zero outside the volume; each intermediate is zeroed outside the
    volume because that is the next layer's padding.  `x` is any array-like
    with numpy slicing (a torch CPU tensor works).  Returns float64."""
    n = ws[0].ndim - 2
    G = tuple(int(g) for g in x.shape[-n:])
    rad = [[(w.shape[2 + i] - 1) // 2 for i in range(n)] for w in ws]
    a = [lo[i] - sum(r[i] for r in rad) for i in range(n)]
    b = [hi[i] + sum(r[i] for r in rad) for i in range(n)]
    lead = tuple(x.shape[:-n])
    cur = np.zeros(lead + tuple(bb - aa for aa, bb in zip(a, b)))
    src = tuple(slice(max(aa, 0), min(bb, g)) for aa, bb, g in zip(a, b, G))
    dst = tuple(slice(s.start - aa, s.stop - aa) for s, aa in zip(src, a))
    piece = x[(Ellipsis,) + src]
    piece = piece.double().numpy() if hasattr(piece, "double") else np.asarray(piece)
    cur[(Ellipsis,) + dst] = piece
    for li, w in enumerate(ws):
        cur = conv_fast(cur, np.asarray(w, dtype=np.float64), 1, 0)
        a = [aa + r for aa, r in zip(a, rad[li])]
        b = [bb - r for bb, r in zip(b, rad[li])]
        if li + 1 < len(ws):
            for i in range(n):
                idx = np.arange(a[i], b[i])
                bad = (idx < 0) | (idx >= G[i])
                if bad.any():
                    sl = [slice(None)] * cur.ndim
                    sl[cur.ndim - n + i] = bad
                    cur[tuple(sl)] = 0.0
    return cur
