"""Hot-path operators: halo convolution and ring attention (fwd + bwd).

Reference: domainpar/ops.py.  Same names, arguments, error types/texts and
collective contracts (halo_conv: exactly 1 collective per rank, empty ranks
included; ring_attention: exactly R-1), registered into the dispatch table
at the reference's levels (ops.py:681-682).  Underneath, every byte of
tensor data is produced by the sm_100a kernels of libdpb200.so:

  halo_conv  = plan (host ints) -> face pack + NCCL send/recv of the right
               halo -> implicit-GEMM conv over the *virtual* extended block
               [local | halo | zeros] (no concatenation, no padding copy)
  backward   = dgrad over the virtual block -> reverse halo (send the halo
               rows' gradient to r+1, accumulate there) -> wgrad partial ->
               all_reduce(dW)
  ring_attention = online-softmax state (m, l, acc) folded block by block
               while K||V circulates (send r+1, recv r-1)
  backward   = (K, V, dK, dV) circulate; one final (dK, dV) hop home

Backward entry points are explicit (`halo_conv_backward`,
`ring_attention_backward`) because collectives must run on the rank's own
thread; `torch.autograd` wrappers (`halo_conv_autograd` / `HaloConv2`,
`ring_attention_autograd` / `RingAttention`) are provided for the
one-process-per-GPU mesh, where they call the same functions.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import kernels
from .dispatch import register_dense_reference, register_handler
from .errors import (DegenerateInputError, DimensionError, HaloError, MetadataError,
                     UnsupportedConfigError)
from .mesh import (AxisGroup, PeerAbort, all_reduce, empty_like_layout, halo_error_text,
                   halo_sendrecv, memory_format_of, ring_shift_known)
from .plan import conv_output_extent, halo_conv_plan, ring_source
from .sharding import Shard, ShardTensor

__all__ = [
    "halo_conv", "halo_conv_forward", "halo_conv_backward", "ConvTape", "dense_conv",
    "ring_attention", "ring_attention_forward", "ring_attention_backward", "AttnTape",
    "sdpa_dense", "RingSoftmaxState", "HaloConv2", "halo_conv_autograd", "RingAttention",
    "ring_attention_autograd",
]


def _group(st: ShardTensor, axis: int) -> AxisGroup:
    return st.ctx.axis_group(st.mesh.axis_names[axis])


def _plain_weight(value, what: str, device) -> torch.Tensor:
    """A plain tensor or a fully replicated ShardTensor (domainpar/ops.py:76-82)."""
    if isinstance(value, ShardTensor):
        if any(isinstance(p, Shard) for p in value.placements):
            raise UnsupportedConfigError(f"{what} must be replicated, not sharded")
        value = value.local
    if not isinstance(value, torch.Tensor):
        value = torch.as_tensor(value)
    if value.device != device:
        value = value.to(device)
    return value


def _conv_params(nsp, kernel, stride, padding):
    """domainpar/dense.py:153-171."""
    strides = (stride,) * nsp if isinstance(stride, int) else tuple(int(s) for s in stride)
    pads = (padding,) * nsp if isinstance(padding, int) else tuple(int(p) for p in padding)
    if len(strides) != nsp or len(pads) != nsp:
        raise DimensionError(f"stride/padding must have one entry per spatial dim ({nsp})")
    for k in kernel:
        if k % 2 != 1:
            raise UnsupportedConfigError(
                f"conv kernels must be odd, got kernel shape {tuple(kernel)}")
    for s in strides:
        if s < 1:
            raise UnsupportedConfigError(f"conv stride must be >= 1, got {s}")
    for p in pads:
        if p < 0:
            raise UnsupportedConfigError(f"conv padding must be >= 0, got {p}")
    return strides, pads


# ---------------------------------------------------------------------------
# dense (single-rank) device references — used for replicated inputs and as
# the dispatch fallback's dense implementations


def dense_conv(x: torch.Tensor, weight: torch.Tensor, stride=1, padding=0) -> torch.Tensor:
    """Cross-correlation, zero padding, dilation 1 (domainpar/dense.py:174-214)
    on one device; x is [C, *sp] or [B, C, *sp]."""
    weight = _plain_weight(weight, "conv weight", x.device)
    nsp = weight.dim() - 2
    if nsp not in (1, 2, 3):
        raise UnsupportedConfigError(
            f"conv supports 1, 2 or 3 spatial dims, weight shape {tuple(weight.shape)} implies "
            f"{nsp}")
    batched = x.dim() == nsp + 2
    if not batched and x.dim() != nsp + 1:
        raise DimensionError(
            f"conv input shape {tuple(x.shape)} incompatible with weight {tuple(weight.shape)}")
    xb = x if batched else x.unsqueeze(0)
    c_out, c_in = weight.shape[:2]
    if xb.shape[1] != c_in:
        raise DimensionError(f"conv input channels {xb.shape[1]} != weight c_in {c_in}")
    kernel = tuple(weight.shape[2:])
    strides, pads = _conv_params(nsp, kernel, stride, padding)
    out_sp = [conv_output_extent(g, k, s, p)
              for g, k, s, p in zip(xb.shape[2:], kernel, strides, pads)]
    w = weight.to(x.dtype).contiguous()
    y = empty_like_layout(xb, [xb.shape[0], c_out] + out_sp)
    kernels.conv_fwd(xb, None, w, y, kernel=kernel, stride=strides,
                     base=[-p for p in pads], shard=-1, halo_rows=0)
    return y if batched else y[0]


def _attn_checks_dense(q, k, v):
    if q.dim() not in (2, 3):
        raise DimensionError(f"q must be [seq, d] or [seq, heads, d], got {tuple(q.shape)}")
    if q.shape[-1] != k.shape[-1] or q.shape[-1] != v.shape[-1]:
        raise DimensionError(f"q/k head dims disagree: {tuple(q.shape)} vs {tuple(k.shape)}")
    if k.shape[0] != v.shape[0]:
        raise DimensionError(f"k/v lengths disagree: {tuple(k.shape)} vs {tuple(v.shape)}")
    if k.shape[0] == 0:
        raise DegenerateInputError("attention over an empty key set")


def sdpa_dense(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """softmax(q k^T / sqrt(d)) v on one device (domainpar/dense.py:258-271)."""
    _attn_checks_dense(q, k, v)
    out, _ = _attn_local(q, [(k, v)], kernels.default_scale(q.shape[-1]))
    return out


# ---------------------------------------------------------------------------
# halo convolution


@dataclass
class ConvTape:
    """What the backward needs from one rank's forward."""

    x: ShardTensor
    weight: torch.Tensor          # [c_out, c_in, *k] in x's dtype, contiguous
    halo: torch.Tensor | None     # right halo rows (batched view)
    plan: object                  # HaloConvPlan or None (unsharded)
    axis: int | None
    d: int | None                 # tensor dim sharded
    sp: int | None                # spatial index sharded
    strides: tuple
    pads: tuple
    batched: bool
    base: tuple                   # per spatial dim window start of output 0
    out: ShardTensor
    xp: torch.Tensor | None = None   # fp32 on the tensor cores: x's bf16x3 parts (split
    xhp: torch.Tensor | None = None  # once in the forward, reused by the weight gradient)


def _validate_conv(x: ShardTensor, weight):
    """All checks the reference runs before any communication
    (domainpar/ops.py:312-361), identically on every rank."""
    weight = _plain_weight(weight, "conv weight", x.local.device)
    nsp = weight.dim() - 2
    if nsp not in (1, 2, 3):
        raise UnsupportedConfigError(
            f"conv supports 1, 2 or 3 spatial dims, weight is {tuple(weight.shape)}")
    batched = x.ndim == nsp + 2
    if not batched and x.ndim != nsp + 1:
        raise DimensionError(
            f"conv input global {x.global_shape} incompatible with weight {tuple(weight.shape)}")
    return weight, nsp, batched


def halo_conv_forward(x: ShardTensor, weight, stride=1, padding=0):
    """Forward halo convolution; returns (out ShardTensor, ConvTape)."""
    weight, nsp, batched = _validate_conv(x, weight)
    first = 2 if batched else 1
    kernel = tuple(weight.shape[2:])
    strides, pads = _conv_params(nsp, kernel, stride, padding)
    sharded = [(axis, p.dim) for axis, p in enumerate(x.placements) if isinstance(p, Shard)]
    xl = x.local
    kernels.require_device("halo_conv", xl)
    w = weight.to(xl.dtype).contiguous()
    xb = xl if batched else xl.unsqueeze(0)
    if not sharded:
        y = dense_conv(xl, w, strides, pads)
        out = ShardTensor(y, tuple(y.shape), x.ctx, x.placements, {})
        tape = ConvTape(x, w, None, None, None, None, None, strides, pads, batched,
                        tuple(-p for p in pads), out)
        return out, tape
    if len(sharded) > 1:
        raise UnsupportedConfigError("halo_conv supports exactly one sharded mesh axis")
    axis, d = sharded[0]
    if d < first:
        raise UnsupportedConfigError(f"halo_conv input is sharded along non-spatial dim {d}")
    sp = d - first
    out_spatial = [conv_output_extent(g, k, s, p)
                   for g, k, s, p in zip(x.global_shape[first:], kernel, strides, pads)]
    c_in = weight.shape[1]
    if x.global_shape[first - 1] != c_in:
        raise DimensionError(
            f"conv input channels {x.global_shape[first - 1]} != weight c_in {c_in}")
    g_in = x.global_shape[d]
    plan = halo_conv_plan(x.shard_shapes[axis], g_in, kernel[sp], strides[sp], pads[sp])
    group = _group(x, axis)
    me = group.index
    mine = plan.members[me]
    # the one exchange round (counted even for empty ranks, ops.py:387)
    x.ctx.collective_count += 1
    bad = plan.hop_violations()
    for requester, width, server, extent in bad:
        if server == me:
            raise HaloError(halo_error_text(group.members[requester], width, x.ctx.rank_id,
                                            extent, d))
    if bad:
        raise PeerAbort(f"rank {x.ctx.rank_id}: unwinding, another rank failed")
    if any(m.lw for m in plan.members):  # cannot happen under anchor ownership
        raise UnsupportedConfigError("halo_conv: left halos are not produced by this ownership")
    serve_left = plan.members[me - 1].rw if me > 0 else 0
    _, halo, pending = halo_sendrecv(group, xb, sp + 2, serve_left, 0, 0, mine.rw, wait=False)
    out_global = tuple(list(x.global_shape[:first - 1]) + [weight.shape[0]] + out_spatial)
    out_sp = list(out_spatial)
    out_sp[sp] = mine.n_out
    base = [-p for p in pads]
    base[sp] = mine.base
    yb = empty_like_layout(xb, [xb.shape[0], weight.shape[0]] + out_sp)
    org = [0] * nsp                       # global index of my output row 0
    org[sp] = sum(plan.out_extents[:me])
    # Interior output rows read only local rows: they are convolved while the
    # halo is in flight; the boundary rows follow once it has landed.
    n_int = _interior_rows(mine.n_out, xb.shape[sp + 2], kernel[sp], strides[sp], mine.base) \
        if mine.rw else mine.n_out
    # fp32 on the tensor cores (bf16x3): split x into its bf16 parts ONCE —
    # both forward launches and the backward's weight gradient read them
    xp = xhp = None
    if yb.numel() and kernels.x3_active(xb, None, yb.shape, yb.stride(), weight.shape[0],
                                        kernel=kernel, stride=strides, base=base, shard=sp,
                                        halo_rows=0):
        xp = kernels.x3_split(xb, kernels.X3_X, kernels.conv_geom(
            xb, None, yb.shape, yb.stride(), weight.shape[0], kernel, strides, base, sp, 0))

    def conv(xh, yv, bb, rows, ob):
        if xp is None:
            kernels.conv_fwd(xb, xh, w, yv, kernel=kernel, stride=strides, base=bb, shard=sp,
                             halo_rows=rows, out_org=ob)
        else:
            kernels.conv_fwd_x3(xb, xh, xp, xhp if rows else None, w, yv, kernel=kernel,
                                stride=strides, base=bb, shard=sp, halo_rows=rows, out_org=ob)

    if yb.numel() and 0 < n_int < mine.n_out:
        conv(None, yb.narrow(sp + 2, 0, n_int), base, 0, org)
    pending.wait()
    if xp is not None and mine.rw:
        xhp = kernels.x3_split(halo, kernels.X3_XHALO, kernels.conv_geom(
            xb, halo, yb.shape, yb.stride(), weight.shape[0], kernel, strides, base, sp, mine.rw))
    if yb.numel() and n_int < mine.n_out:
        bb = list(base)
        bb[sp] = mine.base + n_int * strides[sp]
        ob = list(org)
        ob[sp] += n_int
        conv(halo, yb.narrow(sp + 2, n_int, mine.n_out - n_int), bb, mine.rw, ob)
    elif yb.numel() and n_int == mine.n_out:
        conv(halo, yb, base, mine.rw, org)
    y = yb if batched else yb[0]
    out = ShardTensor(y, out_global, x.ctx, x.placements, {axis: plan.out_extents})
    tape = ConvTape(x, w, halo, plan, axis, d, sp, strides, pads, batched, tuple(base), out,
                    xp, xhp)
    return out, tape


def _interior_rows(n_out: int, extent: int, k: int, s: int, base: int) -> int:
    """Output rows j whose window base + j*s + [0, k) stays inside the
    local block [0, extent) on the sharded dim (a prefix, since base is the
    window start of row 0 and never below the block start for j >= 1 under
    anchor ownership)."""
    if n_out <= 0:
        return 0
    last = extent - k - base  # largest j*s allowed
    if last < 0:
        return 0
    return min(n_out, last // s + 1)


def halo_conv(x: ShardTensor, weight, stride=1, padding=0) -> ShardTensor:
    """Convolution over an input sharded along one spatial dim
    (domainpar/ops.py:303-422): each rank owns the output rows anchored in its
    input interval, fetches its right halo in one exchange round, and
    convolves the virtual extended block.  Handles 1-D/2-D/3-D, uneven and
    empty shards; multi-hop halos raise HaloError on the serving rank."""
    out, _ = halo_conv_forward(x, weight, stride, padding)
    return out


def halo_conv_backward(tape: ConvTape, dout):
    """Gradients of one rank's halo_conv: returns (dx ShardTensor, dW tensor).

    dX_virtual = dgrad(dY) over rows [0, extent + rw) of the virtual block;
    rows [extent, extent + rw) belong to member r+1 and travel back to it
    (one reverse-halo exchange) where they are accumulated into its first
    rows; dW = sum over members of wgrad (one all_reduce).  Two collectives.
    """
    x = tape.x
    dy = dout.local if isinstance(dout, ShardTensor) else dout
    kernels.require_device("halo_conv_backward", dy)
    dyb = dy if tape.batched else dy.unsqueeze(0)
    xl = x.local
    xb = xl if tape.batched else xl.unsqueeze(0)
    w = tape.weight
    kernel = tuple(w.shape[2:])
    wd = kernels.wgrad_dtype(xl.dtype)
    dw = torch.empty(w.shape, dtype=wd, device=xl.device)
    dxb = empty_like_layout(xb, list(xb.shape))
    if tape.plan is None:
        if xb.numel():
            kernels.conv_dgrad(dyb, w, dxb, None, kernel=kernel, stride=tape.strides,
                               base=tape.base, shard=-1, halo_rows=0)
            kernels.conv_wgrad(xb, None, dyb, dw, kernel=kernel, stride=tape.strides,
                               base=tape.base, shard=-1, halo_rows=0)
        else:
            kernels.fill(dw, 0.0)
        dx = dxb if tape.batched else dxb[0]
        return ShardTensor(dx, x.global_shape, x.ctx, x.placements, x.shard_shapes), dw
    group = _group(x, tape.axis)
    me = group.index
    mine = tape.plan.members[me]
    dim = tape.sp + 2
    halo_grad = None
    if mine.rw:
        hshape = list(xb.shape)
        hshape[dim] = mine.rw
        halo_grad = empty_like_layout(xb, hshape)
    work = mine.n_out and xb.shape[dim] + mine.rw
    dyp = None
    if work:
        org = [0] * (xb.dim() - 2)            # global index of my dx row 0
        org[tape.sp] = sum(x.shard_shapes[tape.axis][:me])
        if tape.xp is not None:
            # bf16x3: dy split once, for the data and the weight gradient
            dyp = kernels.x3_split(dyb, kernels.X3_DY, kernels.conv_geom(
                dxb, halo_grad, dyb.shape, dyb.stride(), w.shape[0], kernel, tape.strides,
                tape.base, tape.sp, mine.rw))
            kernels.conv_dgrad_x3(dyb, dyp, w, dxb, halo_grad, kernel=kernel,
                                  stride=tape.strides, base=tape.base, shard=tape.sp,
                                  halo_rows=mine.rw, out_org=org)
        else:
            kernels.conv_dgrad(dyb, w, dxb, halo_grad, kernel=kernel, stride=tape.strides,
                               base=tape.base, shard=tape.sp, halo_rows=mine.rw, out_org=org)
    else:
        kernels.fill(dxb, 0.0)
        kernels.fill(dw, 0.0)
    # reverse halo: my halo rows' gradient goes to r+1, r-1's comes to me;
    # posted before wgrad so the transfer overlaps it
    x.ctx.collective_count += 1
    from_left = tape.plan.members[me - 1].rw if me > 0 else 0
    nxt = group.members[me + 1] if me + 1 < group.size else None
    prv = group.members[me - 1] if me > 0 else None
    sends, recvs = [], []
    if nxt is not None and mine.rw:
        sends.append((nxt, halo_grad))
    incoming = None
    if prv is not None and from_left:
        ishape = list(xb.shape)
        ishape[dim] = from_left
        incoming = empty_like_layout(xb, ishape)
        recvs.append((prv, incoming))
    pending = x.ctx.transport.exchange_start(sends, recvs)
    if work and dyp is not None:
        kernels.conv_wgrad_x3(xb, tape.halo, tape.xp, tape.xhp, dyb, dyp, dw, kernel=kernel,
                              stride=tape.strides, base=tape.base, shard=tape.sp,
                              halo_rows=mine.rw)
    elif work:
        kernels.conv_wgrad(xb, tape.halo, dyb, dw, kernel=kernel, stride=tape.strides,
                           base=tape.base, shard=tape.sp, halo_rows=mine.rw)
    pending.wait()
    if incoming is not None:
        kernels.accumulate(dxb.narrow(dim, 0, from_left), incoming)
    dw = all_reduce(group, dw, "sum")
    dx = dxb if tape.batched else dxb[0]
    return ShardTensor(dx, x.global_shape, x.ctx, x.placements, x.shard_shapes), dw


# ---------------------------------------------------------------------------
# ring attention


class RingSoftmaxState:
    """Device-resident online-softmax accumulator (domainpar/ops.py:180-214):
    running row max m, denominator l, numerator acc — fp64 for fp32/fp64
    inputs (as the reference), fp32 for bf16.  `update` folds one score/value
    block through the attention-block kernel; any block order gives the same
    output up to rounding."""

    def __init__(self, rows: int, heads: int, dim: int, dtype: torch.dtype, device):
        sd = kernels.state_dtype(dtype)
        self.m = kernels.fill(torch.empty((rows, heads), dtype=sd, device=device), -math.inf)
        self.l = kernels.zeros((rows, heads), sd, device)
        self.acc = kernels.zeros((rows, heads, dim), sd, device)

    def update(self, q, k, v, scale) -> None:
        if k.shape[0] == 0 or q.shape[0] == 0:
            return
        kernels.attn_fwd_update(q, k, v, self.m, self.l, self.acc, scale)

    def output(self, q, out_dtype) -> tuple:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
        lse = torch.empty(self.m.shape, dtype=self.m.dtype, device=q.device)
        if q.shape[0]:
            kernels.attn_finalize(q, self.m, self.l, self.acc, out, lse, 1.0)
        return out, lse


def _attn_local(q, blocks, scale):
    """Fold (k, v) blocks into a fresh state on one device; returns (out, lse)."""
    heads = q.shape[1] if q.dim() == 3 else 1
    state = RingSoftmaxState(q.shape[0], heads, q.shape[-1], q.dtype, q.device)
    for k, v in blocks:
        state.update(q, k, v, scale)
    return state.output(q, q.dtype)


@dataclass
class AttnTape:
    q: ShardTensor
    k: ShardTensor
    v: ShardTensor
    out: ShardTensor
    lse: torch.Tensor
    axis: int | None
    scale: float


def _check_attention(q, k, v):
    """domainpar/ops.py:226-264 (2-D [seq, d]; 3-D [seq, heads, d] added)."""
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not isinstance(t, ShardTensor):
            raise TypeError(f"ring_attention {name} must be a ShardTensor")
        if t.ndim not in (2, 3):
            raise DimensionError(
                f"ring_attention {name} must be [seq, head_dim] or [seq, heads, head_dim], "
                f"global is {t.global_shape}")
        for dim in range(1, t.ndim):
            if t.sharded_axis_for_dim(dim) is not None:
                raise UnsupportedConfigError(f"ring_attention {name} has a sharded head dim")
    if k.ctx is not q.ctx or v.ctx is not q.ctx:
        raise MetadataError("ring_attention operands live on different mesh runs")
    if q.ndim != k.ndim or q.ndim != v.ndim or q.global_shape[1:-1] != k.global_shape[1:-1] \
            or k.global_shape[1:-1] != v.global_shape[1:-1]:
        raise DimensionError(f"head layouts disagree: q {q.global_shape}, k {k.global_shape}, "
                             f"v {v.global_shape}")
    d = q.global_shape[-1]
    if k.global_shape[-1] != d or v.global_shape[-1] != d:
        raise DimensionError(f"head dims disagree: q {q.global_shape}, k {k.global_shape}, "
                             f"v {v.global_shape}")
    if k.global_shape[0] != v.global_shape[0]:
        raise DimensionError(f"k/v lengths disagree: {k.global_shape} vs {v.global_shape}")
    if k.global_shape[0] == 0:
        raise DegenerateInputError("ring_attention over an empty key set")
    qa, ka, va = (t.sharded_axis_for_dim(0) for t in (q, k, v))
    if ka != va or k.shard_shapes != v.shard_shapes:
        raise MetadataError("k and v must share one sequence sharding")
    if qa != ka:
        raise MetadataError("q and k/v must be sequence-sharded on the same mesh axis")
    return qa


def _kv_payload(k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """K and V ride one contiguous payload [S, 2, H, d] (domainpar/ops.py:270
    concatenates them as [S, 2d]); K = payload[:, 0], V = payload[:, 1]."""
    k3 = k.unsqueeze(1) if k.dim() == 2 else k
    v3 = v.unsqueeze(1) if v.dim() == 2 else v
    pay = torch.empty((k3.shape[0], 2) + tuple(k3.shape[1:]), dtype=k.dtype, device=k.device)
    if pay.numel():
        kernels.copy_strided(pay[:, 0], k3)
        kernels.copy_strided(pay[:, 1], v3)
    return pay


def ring_attention_forward(q: ShardTensor, k: ShardTensor, v: ShardTensor):
    """Forward ring attention; returns (out ShardTensor, AttnTape)."""
    qa = _check_attention(q, k, v)
    d = q.global_shape[-1]
    scale = 1.0 / math.sqrt(d)
    kernels.require_device("ring_attention", q.local, k.local, v.local)
    if qa is None:
        out, lse = _attn_local(q.local, [(k.local, v.local)], scale)
        res = ShardTensor(out, q.global_shape, q.ctx, q.placements, q.shard_shapes)
        return res, AttnTape(q, k, v, res, lse, None, scale)
    group = _group(q, qa)
    r, me = group.size, group.index
    kv_ext = k.shard_shapes[qa]
    ql = q.local
    heads = ql.shape[1] if ql.dim() == 3 else 1
    state = RingSoftmaxState(ql.shape[0], heads, d, ql.dtype, ql.device)
    pay = _kv_payload(k.local, v.local)
    for step in range(r):
        # the next K||V hop is posted before this block's attention kernel, so
        # the transfer over NVLink overlaps the compute (double-buffered)
        nxt_pay = pending = None
        if step < r - 1:
            q.ctx.collective_count += 1
            src = ring_source(me, step + 1, r)
            nxt_pay, pending = _ring_post(group, pay, (kv_ext[src],) + tuple(pay.shape[1:]))
        if pay.shape[0]:
            kb, vb = pay[:, 0], pay[:, 1]
            if ql.dim() == 2:
                kb, vb = kb[:, 0], vb[:, 0]
            state.update(ql, kb, vb, scale)
        if pending is not None:
            pending.wait()
            pay = nxt_pay
    out, lse = state.output(ql, ql.dtype)
    res = ShardTensor(out, q.global_shape, q.ctx, q.placements, q.shard_shapes)
    return res, AttnTape(q, k, v, res, lse, qa, scale)


def _ring_post(group: AxisGroup, payload: torch.Tensor, recv_shape):
    """Post one ring hop (send to index+1, receive `recv_shape` from
    index-1) and return (receive buffer, handle); R = 1 never posts."""
    r = group.size
    nxt = group.members[(group.index + 1) % r]
    prv = group.members[(group.index - 1) % r]
    out = torch.empty(tuple(recv_shape), dtype=payload.dtype, device=payload.device)
    sends = [(nxt, payload.contiguous())] if payload.numel() else []
    recvs = [(prv, out)] if out.numel() else []
    if group.ctx.transport.kind == "thread":
        # per-pair FIFO mailboxes: empty payloads still travel (pairing never
        # depends on the data)
        sends = [(nxt, payload.contiguous())]
        recvs = [(prv, out)]
    return out, group.ctx.transport.exchange_start(sends, recvs)


def ring_attention(q: ShardTensor, k: ShardTensor, v: ShardTensor) -> ShardTensor:
    """Sequence-sharded attention with K/V circulating the group
    (domainpar/ops.py:217-279): exactly R-1 ring shifts, one K||V payload per
    shift, online softmax that never materialises the score matrix.  q may be
    sharded differently from k/v; empty shards still shift."""
    out, _ = ring_attention_forward(q, k, v)
    return out


def ring_attention_backward(tape: AttnTape, dout):
    """Gradients (dq, dk, dv) as ShardTensors with the inputs' layouts.

    With P = exp(q k^T scale - lse), D = rowsum(dO * O): dV += P^T dO,
    dS = P (dO V^T - D), dQ += scale dS K, dK += scale dS^T Q.  K, V and their
    dK/dV accumulators circulate together (R-1 shifts), then one final hop
    returns each dK/dV block to its owner: R collectives."""
    q, k, v = tape.q, tape.k, tape.v
    do = dout.local if isinstance(dout, ShardTensor) else dout
    ql, ol = q.local, tape.out.local
    kernels.require_device("ring_attention_backward", do)
    sd = kernels.state_dtype(ql.dtype)
    heads = ql.shape[1] if ql.dim() == 3 else 1
    d = ql.shape[-1]
    delta = torch.empty((ql.shape[0], heads), dtype=sd, device=ql.device)
    if ql.shape[0]:
        kernels.attn_bwd_preprocess(ol, do, delta)
    dq = kernels.zeros((ql.shape[0], heads, d), sd, ql.device)

    def run_block(kb, vb, dkb, dvb):
        if kb.shape[0] == 0 or ql.shape[0] == 0:
            return
        kernels.attn_bwd_update(ql, kb, vb, do, tape.lse, delta, dq, dkb, dvb, tape.scale)

    if tape.axis is None:
        kl, vl = k.local, v.local
        dk = kernels.zeros((kl.shape[0], heads, d), sd, ql.device)
        dv = kernels.zeros((kl.shape[0], heads, d), sd, ql.device)
        run_block(kl, vl, dk, dv)
    else:
        group = _group(q, tape.axis)
        r, me = group.size, group.index
        kv_ext = k.shard_shapes[tape.axis]
        pay = _kv_payload(k.local, v.local)
        # dK and dV accumulators travel as one contiguous [2, S, H, d] payload.
        # K||V hops are posted before each block's kernel (overlapped); the
        # block's own contribution is computed into a fresh accumulator while
        # the partial sums of the previous members are still in flight, and
        # the two are added before the sum moves on.
        incoming = pending_g = None
        grads = None
        for step in range(r):
            src_now = ring_source(me, step, r)
            nxt_pay = pending = None
            if step < r - 1:
                q.ctx.collective_count += 1
                src = ring_source(me, step + 1, r)
                nxt_pay, pending = _ring_post(group, pay, (kv_ext[src],) + tuple(pay.shape[1:]))
            grads = kernels.zeros((2, kv_ext[src_now], heads, d), sd, ql.device)
            if pay.shape[0]:
                kb, vb = pay[:, 0], pay[:, 1]
                if ql.dim() == 2:
                    kb, vb = kb[:, 0], vb[:, 0]
                run_block(kb, vb, grads[0], grads[1])
            if pending_g is not None:
                pending_g.wait()
                if grads.numel():
                    kernels.accumulate(grads, incoming)
            if step < r - 1:
                incoming, pending_g = _ring_post(group, grads,
                                                 (2, kv_ext[ring_source(me, step + 1, r)], heads, d))
            if pending is not None:
                pending.wait()
                pay = nxt_pay
        if r > 1:
            # block held now is member (me - (r-1)) mod r = me + 1: one hop home
            q.ctx.collective_count += 1
            grads = ring_shift_known(group, grads, (2, kv_ext[me], heads, d))
        dk, dv = grads[0], grads[1]

    def finish(acc, like: ShardTensor):
        t = acc if like.local.dim() == 3 else acc[:, 0]
        out = torch.empty(like.local.shape, dtype=like.local.dtype, device=like.local.device)
        if out.numel():
            _cast_into(out, t)
        return ShardTensor(out, like.global_shape, like.ctx, like.placements, like.shard_shapes)

    return finish(dq, q), finish(dk, k), finish(dv, v)


def _cast_into(dst: torch.Tensor, src: torch.Tensor) -> None:
    """Accumulator -> parameter dtype (dp_convert_strided: one HBM pass)."""
    kernels.convert(dst, src)


# ---------------------------------------------------------------------------
# autograd wrappers (one process per GPU)


class HaloConv2(torch.autograd.Function):
    """torch.autograd bridge for halo_conv on a process mesh."""

    @staticmethod
    def forward(actx, x_local, weight, xst, stride, padding):
        st = ShardTensor(x_local.detach(), xst.global_shape, xst.ctx, xst.placements,
                         xst.shard_shapes)
        out, tape = halo_conv_forward(st, weight.detach(), stride, padding)
        actx.tape = tape
        actx.wdtype = weight.dtype
        actx.out_fmt = memory_format_of(out.local)
        return out.local

    @staticmethod
    def backward(actx, gy):
        dx, dw = halo_conv_backward(actx.tape, gy.contiguous(memory_format=actx.out_fmt))
        return dx.local, dw.to(actx.wdtype), None, None, None


def _need_process_mesh(ctx, what: str) -> None:
    if ctx.transport.kind == "thread":
        raise UnsupportedConfigError(
            f"autograd through collectives needs one process per rank; use "
            f"{what}_forward/{what}_backward on a thread mesh")


def halo_conv_autograd(x: ShardTensor, weight, stride=1, padding=0) -> ShardTensor:
    """halo_conv whose `.local` carries a grad_fn (process meshes only).
    `weight` is a plain tensor or a fully replicated ShardTensor (its local
    tensor is the autograd leaf, as domainpar/ops.py:76-82 accepts both)."""
    _need_process_mesh(x.ctx, "halo_conv")
    weight_p = _plain_weight(weight, "conv weight", x.local.device)
    y = HaloConv2.apply(x.local, weight_p, x, stride, padding)
    nsp = weight_p.dim() - 2
    first = 2 if x.ndim == nsp + 2 else 1
    kernel = tuple(weight_p.shape[2:])
    strides, pads = _conv_params(nsp, kernel, stride, padding)
    out_spatial = [conv_output_extent(g, kk, s, p)
                   for g, kk, s, p in zip(x.global_shape[first:], kernel, strides, pads)]
    out_global = tuple(list(x.global_shape[:first - 1]) + [weight_p.shape[0]] + out_spatial)
    shapes = {}
    for axis, p in enumerate(x.placements):
        if isinstance(p, Shard):
            sp = p.dim - first
            plan = halo_conv_plan(x.shard_shapes[axis], x.global_shape[p.dim], kernel[sp],
                                  strides[sp], pads[sp])
            shapes[axis] = plan.out_extents
    return ShardTensor(y, out_global, x.ctx, x.placements, shapes)


class RingAttention(torch.autograd.Function):
    """torch.autograd bridge for ring_attention on a process mesh: forward =
    ring_attention_forward, backward = ring_attention_backward (the (K, V,
    dK, dV) ring plus the final hop home)."""

    @staticmethod
    def forward(actx, q_local, k_local, v_local, qst, kst, vst):
        def st(t, like):
            return ShardTensor(t.detach(), like.global_shape, like.ctx, like.placements,
                               like.shard_shapes)

        out, tape = ring_attention_forward(st(q_local, qst), st(k_local, kst), st(v_local, vst))
        actx.tape = tape
        return out.local

    @staticmethod
    def backward(actx, go):
        dq, dk, dv = ring_attention_backward(actx.tape, go.contiguous())
        return dq.local, dk.local, dv.local, None, None, None


def ring_attention_autograd(q: ShardTensor, k: ShardTensor, v: ShardTensor) -> ShardTensor:
    """ring_attention whose `.local` carries a grad_fn (process meshes only);
    gradients flow to q.local, k.local and v.local."""
    _need_process_mesh(q.ctx, "ring_attention")
    y = RingAttention.apply(q.local, k.local, v.local, q, k, v)
    return ShardTensor(y, q.global_shape, q.ctx, q.placements, q.shard_shapes)


# ---------------------------------------------------------------------------
# default registrations (domainpar/ops.py:674-696)

register_handler("aten_like", "conv", halo_conv)
register_handler("named_function", "ring_attention", ring_attention)
register_dense_reference("conv", dense_conv)
register_dense_reference("sdpa", sdpa_dense)
register_dense_reference("ring_attention", sdpa_dense)
