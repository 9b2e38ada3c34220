"""The operators around the hot path: pointwise
and linear ops, the sharded normalisations, data-parallel gradient
averaging and the ViT patch-tokenizer + transformer-block pipeline.

Reference: domainpar/ops.py:93-173 (sharded_elementwise / _linear /
_softmax / _layer_norm), :429-444 (ddp_allreduce_grads), :447-655 (VitConfig,
make_vit_weights, image_to_sequence, vit_block_pipeline(_dense)),
domainpar/dense.py:54-116, :223-255 (the dense twins), domainpar/memory.py:
270-296 (ActivationLedger).  Same names, arguments, error types/texts and
collective counts (elementwise / linear: 0; layer_norm: 1 — both moments
ride one stacked all_reduce; softmax: 2 — max, then denominator).

Device work: statistics, normalisation and pointwise math are the sm_100a
kernels of libdpb200.so (dp_norm_stats / dp_norm_apply / dp_elementwise,
fp64 statistics like the reference); `linear` is a plain library GEMM
(cuBLAS through torch.addmm).  One deliberate change:
vit_block_pipeline runs ONE ring over all heads ([seq, heads, head_dim]
views of q/k/v) instead of one ring per head, so a layer costs R-1 K||V
hops instead of n_heads*(R-1); the dense twin and the per-head reference
agree to rounding.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from .dispatch import dispatch_operation, register_dense_reference, register_handler
from .errors import (DegenerateInputError, DimensionError, MetadataError,
                     UnsupportedConfigError)
from .mesh import AxisGroup, all_reduce
from .ops import dense_conv, sdpa_dense
from .sharding import Shard, ShardTensor

__all__ = [
    "ELEMENTWISE_OPS", "dense_elementwise", "dense_add", "dense_mul", "dense_scale",
    "dense_matmul", "dense_linear", "dense_softmax", "dense_layer_norm",
    "sharded_elementwise", "sharded_linear", "sharded_softmax", "sharded_layer_norm",
    "ddp_allreduce_grads", "image_to_sequence", "ActivationLedger", "VitConfig",
    "make_vit_weights", "vit_block_pipeline", "vit_block_pipeline_dense",
]

ELEMENTWISE_OPS = ("add", "mul", "scale")
_EW = {"add": _lib.EW_ADD, "mul": _lib.EW_MUL, "scale": _lib.EW_SCALE}


def _normalize_dim(dim: int, ndim: int) -> int:
    """domainpar/ops.py:85-88."""
    if not -ndim <= dim < ndim:
        raise DimensionError(f"axis {dim} out of range for rank-{ndim} tensor")
    return dim % ndim


def _group_for_axis(st: ShardTensor, axis: int) -> AxisGroup:
    return st.ctx.axis_group(st.mesh.axis_names[axis])


def _plain(value, what: str, device) -> torch.Tensor:
    """A plain tensor/array or a fully replicated ShardTensor (ops.py:76-82)."""
    if isinstance(value, ShardTensor):
        if any(isinstance(p, Shard) for p in value.placements):
            raise UnsupportedConfigError(f"{what} must be replicated, not sharded")
        value = value.local
    if not isinstance(value, torch.Tensor):
        value = torch.as_tensor(np.asarray(value))
    return value.to(device) if value.device != device else value


def _require_same_layout(what: str, a: ShardTensor, b: ShardTensor) -> None:
    """domainpar/ops.py:63-73."""
    if a.ctx is not b.ctx:
        raise MetadataError(f"{what}: operands live on different mesh runs")
    if tuple(a.global_shape) != tuple(b.global_shape):
        raise DimensionError(
            f"{what}: global shapes disagree: {tuple(a.global_shape)} vs "
            f"{tuple(b.global_shape)}")
    if tuple(a.placements) != tuple(b.placements) or a.shard_shapes != b.shard_shapes:
        raise MetadataError(
            f"{what}: operand layouts disagree: {list(a.placements)}/{a.shard_shapes} vs "
            f"{list(b.placements)}/{b.shard_shapes}")


# ---------------------------------------------------------------------------
# dense (one-device) twins: domainpar/dense.py


def _is_scalar(b) -> bool:
    if isinstance(b, torch.Tensor):
        return b.dim() == 0
    if isinstance(b, np.ndarray):
        return b.ndim == 0
    return isinstance(b, (int, float, np.number))


def dense_elementwise(op: str, a: torch.Tensor, b) -> torch.Tensor:
    """add / mul / scale with no broadcasting: shapes match exactly, or b is
    a scalar (domainpar/dense.py:65-98)."""
    if op not in _EW:
        raise UnsupportedConfigError(
            f"unknown elementwise op {op!r}; expected one of {ELEMENTWISE_OPS}")
    if op == "scale":
        if not _is_scalar(b):
            shape = tuple(b.shape) if hasattr(b, "shape") else ()
            raise DimensionError(f"scale expects a scalar, got array of shape {shape}")
        return kernels.elementwise(_lib.EW_SCALE, a, scalar=float(b))
    if _is_scalar(b):
        return kernels.elementwise(_EW[op], a, scalar=float(b))
    b = _plain(b, f"{op} operand", a.device)
    if tuple(a.shape) != tuple(b.shape):
        raise DimensionError(
            f"{op} operand shapes disagree: {tuple(a.shape)} vs {tuple(b.shape)}")
    return kernels.elementwise(_EW[op], a, b)


def dense_add(a, b):
    return dense_elementwise("add", a, b)


def dense_mul(a, b):
    return dense_elementwise("mul", a, b)


def dense_scale(a, s):
    return dense_elementwise("scale", a, s)


def _check_2d(name: str, a: torch.Tensor) -> None:
    if a.dim() != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {tuple(a.shape)}")


def dense_matmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """[m,k] @ [k,n] (domainpar/dense.py:54-62), cuBLAS."""
    _check_2d("a", a)
    _check_2d("b", b)
    if a.shape[1] != b.shape[0]:
        raise DimensionError(
            f"matmul inner dims disagree: a is {tuple(a.shape)}, b is {tuple(b.shape)}")
    return a @ b.to(a.dtype)


def dense_linear(x: torch.Tensor, weight, bias) -> torch.Tensor:
    """z = x @ W^T + b (domainpar/dense.py:101-116); a plain cuBLAS GEMM."""
    weight = _plain(weight, "linear weight", x.device)
    bias = _plain(bias, "linear bias", x.device)
    _check_2d("x", x)
    _check_2d("weight", weight)
    if bias.dim() != 1:
        raise DimensionError(f"bias must be 1-D, got shape {tuple(bias.shape)}")
    n_out, n_in = weight.shape
    if x.shape[1] != n_in:
        raise DimensionError(
            f"linear input width {x.shape[1]} does not match weight n_in {n_in}")
    if bias.shape[0] != n_out:
        raise DimensionError(
            f"bias length {bias.shape[0]} does not match weight n_out {n_out}")
    kernels.require_device("linear", x)
    return torch.addmm(bias.to(x.dtype), x, weight.to(x.dtype).t())


def _check_axis(x: torch.Tensor, dim: int) -> int:
    if not -x.dim() <= dim < x.dim():
        raise DimensionError(f"axis {dim} out of range for shape {tuple(x.shape)}")
    return dim % x.dim()


def dense_softmax(x: torch.Tensor, dim: int) -> torch.Tensor:
    """Max-shifted softmax in fp64 statistics (domainpar/dense.py:223-234)."""
    dim = _check_axis(x, dim)
    if x.shape[dim] == 0:
        raise DegenerateInputError(
            f"softmax over zero-extent axis {dim} of shape {tuple(x.shape)}")
    x = kernels.contiguous(x)
    gmax = kernels.norm_stats(_lib.NORM_MAX, x, dim)
    den = kernels.norm_stats(_lib.NORM_EXPSUM, x, dim, aux=gmax)
    return kernels.norm_apply(1, x, dim, den, gmax, 1.0)


def dense_layer_norm(x: torch.Tensor, dim: int, eps: float = 1e-5) -> torch.Tensor:
    """Population layer norm from fp64 moments (domainpar/dense.py:237-255)."""
    dim = _check_axis(x, dim)
    n = x.shape[dim]
    if n == 0:
        raise DegenerateInputError(
            f"layer_norm over zero-extent axis {dim} of shape {tuple(x.shape)}")
    x = kernels.contiguous(x)
    sums = kernels.norm_stats(_lib.NORM_MOMENTS, x, dim)
    return kernels.norm_apply(0, x, dim, sums, None, float(n), eps)


# ---------------------------------------------------------------------------
# sharded ops: domainpar/ops.py:93-173


def sharded_elementwise(op: str, a: ShardTensor, b) -> ShardTensor:
    """add/mul/scale on matching layouts (or a scalar b).  Pure local."""
    if not isinstance(a, ShardTensor):
        raise TypeError("sharded_elementwise expects a ShardTensor first operand")
    if isinstance(b, ShardTensor):
        _require_same_layout(f"elementwise {op}", a, b)
        local = dense_elementwise(op, a.local, b.local)
    else:
        local = dense_elementwise(op, a.local, b)
    return ShardTensor(local, a.global_shape, a.ctx, a.placements, a.shard_shapes)


def sharded_linear(x: ShardTensor, weight, bias) -> ShardTensor:
    """x @ W^T + b with x [rows, n_in]; rows may be sharded, n_in may not."""
    weight = _plain(weight, "linear weight", x.local.device)
    bias = _plain(bias, "linear bias", x.local.device)
    if x.ndim != 2:
        raise DimensionError(f"linear input must be 2-D, global is {tuple(x.global_shape)}")
    if x.sharded_axis_for_dim(1) is not None:
        raise UnsupportedConfigError(
            "linear contraction dim (1) is sharded; gather or redistribute first")
    local = dense_linear(x.local, weight, bias)
    out_global = (x.global_shape[0], weight.shape[0])
    return ShardTensor(local, out_global, x.ctx, x.placements, x.shard_shapes)


def sharded_softmax(x: ShardTensor, dim: int) -> ShardTensor:
    """Softmax along dim; aggregates max and denominator across the shards
    (two all_reduces)."""
    dim = _normalize_dim(dim, x.ndim)
    if x.global_shape[dim] == 0:
        raise DegenerateInputError(
            f"softmax over zero-extent dim {dim} of global {tuple(x.global_shape)}")
    axis = x.sharded_axis_for_dim(dim)
    if axis is None:
        local = dense_softmax(x.local, dim) if x.local.numel() else x.local.clone()
        return ShardTensor(local, x.global_shape, x.ctx, x.placements, x.shard_shapes)
    group = _group_for_axis(x, axis)
    xl = kernels.contiguous(x.local)
    kernels.require_device("softmax", xl)
    gmax = all_reduce(group, kernels.norm_stats(_lib.NORM_MAX, xl, dim), op="max")
    denom = all_reduce(group, kernels.norm_stats(_lib.NORM_EXPSUM, xl, dim, aux=gmax), op="sum")
    out = kernels.norm_apply(1, xl, dim, denom, gmax, 1.0)
    return ShardTensor(out, x.global_shape, x.ctx, x.placements, x.shard_shapes)


def sharded_layer_norm(x: ShardTensor, dim: int, eps: float = 1e-5) -> ShardTensor:
    """Normalize along dim using all-reduced float64 moments (ONE all_reduce:
    sum and sum of squares ride one [2, cells] buffer)."""
    dim = _normalize_dim(dim, x.ndim)
    n = x.global_shape[dim]
    if n == 0:
        raise DegenerateInputError(
            f"layer_norm over zero-extent dim {dim} of global {tuple(x.global_shape)}")
    axis = x.sharded_axis_for_dim(dim)
    if axis is None:
        local = dense_layer_norm(x.local, dim, eps) if x.local.numel() else x.local.clone()
        return ShardTensor(local, x.global_shape, x.ctx, x.placements, x.shard_shapes)
    group = _group_for_axis(x, axis)
    xl = kernels.contiguous(x.local)
    kernels.require_device("layer_norm", xl)
    sums = all_reduce(group, kernels.norm_stats(_lib.NORM_MOMENTS, xl, dim), op="sum")
    out = kernels.norm_apply(0, xl, dim, sums, None, float(n), eps)
    return ShardTensor(out, x.global_shape, x.ctx, x.placements, x.shard_shapes)


# ---------------------------------------------------------------------------
# data-parallel gradient averaging: domainpar/ops.py:429-444


def ddp_allreduce_grads(group: AxisGroup, grads):
    """Average each gradient across the group (one all_reduce per tensor).
    Accepts a list/tuple or a name->tensor dict and returns the same
    container type; the sum is folded in member order, then scaled by
    1/size on every rank."""
    inv = 1.0 / group.size

    def mean_of(g):
        g = g if isinstance(g, torch.Tensor) else torch.as_tensor(np.asarray(g))
        if group.ctx.device.type == "cuda" and not g.is_cuda:
            g = g.to(group.ctx.device)
        return kernels.elementwise(_lib.EW_SCALE, all_reduce(group, g, op="sum"), scalar=inv)

    if isinstance(grads, dict):
        return {name: mean_of(g) for name, g in grads.items()}
    out = [mean_of(g) for g in grads]
    return tuple(out) if isinstance(grads, tuple) else out


# ---------------------------------------------------------------------------
# ViT pipeline: domainpar/ops.py:447-655, domainpar/memory.py:270-296


class ActivationLedger:
    """Byte counter for saved activations (peak == total: nothing is
    released before the hypothetical backward)."""

    def __init__(self):
        self.total_bytes = 0
        self.n_saved = 0

    def save(self, value) -> None:
        if isinstance(value, ShardTensor):
            value = value.local
        if isinstance(value, torch.Tensor):
            nbytes = value.numel() * value.element_size()
        elif isinstance(value, np.ndarray):
            nbytes = value.nbytes
        else:
            nbytes = int(value)
        if nbytes < 0:
            raise UnsupportedConfigError(f"negative byte count {nbytes}")
        self.total_bytes += nbytes
        self.n_saved += 1

    @property
    def peak_bytes(self) -> int:
        return self.total_bytes

    def reset(self) -> None:
        self.total_bytes = 0
        self.n_saved = 0


@dataclass(frozen=True)
class VitConfig:
    """Shapes for the patch-tokenizer + transformer-block pipeline."""

    image_channels: int = 3
    patch: int = 5  # tokenizer kernel == stride; odd so the conv contract holds
    embed_dim: int = 64
    n_layers: int = 16
    n_heads: int = 4
    mlp_ratio: int = 4
    eps: float = 1e-5

    def __post_init__(self):
        if self.patch % 2 != 1:
            raise UnsupportedConfigError(f"patch must be odd, got {self.patch}")
        if self.embed_dim % self.n_heads != 0:
            raise UnsupportedConfigError(
                f"embed_dim {self.embed_dim} not divisible by n_heads {self.n_heads}")
        if min(self.image_channels, self.embed_dim, self.n_heads,
               self.mlp_ratio) < 1 or self.n_layers < 0:
            raise UnsupportedConfigError("VitConfig fields must be positive")

    @property
    def head_dim(self) -> int:
        return self.embed_dim // self.n_heads

    @property
    def mlp_hidden(self) -> int:
        return self.embed_dim * self.mlp_ratio


def make_vit_weights(config: VitConfig, seed: int = 0, dtype=torch.float32,
                     device=None) -> dict:
    """Seeded weights for vit_block_pipeline: the same NumPy draws as the
    reference (domainpar/ops.py:485-510), so both frameworks share every
    parameter bit; returned as torch tensors on `device`."""
    rng = np.random.default_rng(seed)
    d, h = config.embed_dim, config.mlp_hidden
    np_dtype = np.float64 if dtype == torch.float64 else np.float32

    def w(*shape):
        arr = (rng.standard_normal(shape) * 0.05).astype(np_dtype)
        t = torch.from_numpy(arr).to(dtype)
        return t.to(device) if device is not None else t

    weights = {"tokenizer": w(d, config.image_channels, config.patch, config.patch)}
    for i in range(config.n_layers):
        for name, shape in (("wq", (d, d)), ("bq", (d,)), ("wk", (d, d)), ("bk", (d,)),
                            ("wv", (d, d)), ("bv", (d,)), ("wo", (d, d)), ("bo", (d,)),
                            ("w1", (h, d)), ("b1", (h,)), ("w2", (d, h)), ("b2", (d,))):
            weights[f"layers.{i}.{name}"] = w(*shape)
    return weights


def image_to_sequence(t: ShardTensor) -> ShardTensor:
    """[channels, h, w] -> [h*w, channels] token sequence, purely local; a
    shard along h becomes a shard along tokens with extents h_r * w."""
    if t.ndim != 3:
        raise DimensionError(f"expected [channels, h, w], global {tuple(t.global_shape)}")
    c, h, w = t.global_shape
    axis = t.sharded_axis_for_dim(1)
    if t.sharded_axis_for_dim(0) is not None or t.sharded_axis_for_dim(2) is not None:
        raise UnsupportedConfigError("image_to_sequence supports sharding along h only")
    local = kernels.contiguous(t.local.permute(1, 2, 0)).reshape(-1, c)
    if axis is None:
        placements, shapes = t.placements, {}
    else:
        placements = tuple(Shard(0) if isinstance(p, Shard) else p for p in t.placements)
        shapes = {axis: tuple(e * w for e in t.shard_shapes[axis])}
    return ShardTensor(local, (h * w, c), t.ctx, placements, shapes)


def _heads_view(t: ShardTensor, n_heads: int) -> ShardTensor:
    """[tokens, heads*dh] -> [tokens, heads, dh] (a view; same sharding)."""
    s, d = t.global_shape
    local = t.local.view(t.local.shape[0], n_heads, d // n_heads)
    return ShardTensor(local, (s, n_heads, d // n_heads), t.ctx, t.placements, t.shard_shapes)


def _merge_heads(t: ShardTensor) -> ShardTensor:
    s, hh, dh = t.global_shape
    local = t.local.reshape(t.local.shape[0], hh * dh)
    return ShardTensor(local, (s, hh * dh), t.ctx, t.placements, t.shard_shapes)


def vit_block_pipeline(x: ShardTensor, config: VitConfig, weights,
                       ledger: ActivationLedger | None = None, table=None) -> ShardTensor:
    """Patch tokenizer + n_layers transformer blocks, domain-parallel
    (domainpar/ops.py:559-612).  x is one sample [channels, h, w] sharded
    along h; the tokenizer conv runs under halo exchange, tokens stay
    sequence-sharded, attention rides ONE ring for all heads, layer norms are
    over the whole embedding dim.  Returns the [tokens, embed_dim] sequence."""
    def save(t):
        if ledger is not None:
            ledger.save(t)

    def op(name, *args, **kwargs):
        return dispatch_operation(name, *args, table=table, **kwargs)

    save(x)
    tokens = op("conv", x, weights["tokenizer"], stride=config.patch, padding=0)
    seq = image_to_sequence(tokens)
    for i in range(config.n_layers):
        p = f"layers.{i}."
        save(seq)
        normed = op("layer_norm", seq, 1, eps=config.eps)
        save(normed)
        q = op("linear", normed, weights[p + "wq"], weights[p + "bq"])
        k = op("linear", normed, weights[p + "wk"], weights[p + "bk"])
        v = op("linear", normed, weights[p + "wv"], weights[p + "bv"])
        save(q), save(k), save(v)
        attn = _merge_heads(op("ring_attention", _heads_view(q, config.n_heads),
                               _heads_view(k, config.n_heads), _heads_view(v, config.n_heads)))
        save(attn)
        proj = op("linear", attn, weights[p + "wo"], weights[p + "bo"])
        seq = op("add", seq, proj)
        save(seq)
        normed2 = op("layer_norm", seq, 1, eps=config.eps)
        save(normed2)
        hidden = op("linear", normed2, weights[p + "w1"], weights[p + "b1"])
        save(hidden)
        mlp = op("linear", hidden, weights[p + "w2"], weights[p + "b2"])
        seq = op("add", seq, mlp)
    return seq


def vit_block_pipeline_dense(x: torch.Tensor, config: VitConfig, weights,
                             ledger: ActivationLedger | None = None) -> torch.Tensor:
    """Single-device twin of vit_block_pipeline (domainpar/ops.py:615-655)."""
    def save(t):
        if ledger is not None:
            ledger.save(t)

    save(x)
    tokens = dense_conv(x, weights["tokenizer"], stride=config.patch, padding=0)
    c = tokens.shape[0]
    seq = kernels.contiguous(tokens.permute(1, 2, 0)).reshape(-1, c)
    hh, dh = config.n_heads, config.head_dim
    for i in range(config.n_layers):
        p = f"layers.{i}."
        save(seq)
        normed = dense_layer_norm(seq, 1, eps=config.eps)
        save(normed)
        q = dense_linear(normed, weights[p + "wq"], weights[p + "bq"])
        k = dense_linear(normed, weights[p + "wk"], weights[p + "bk"])
        v = dense_linear(normed, weights[p + "wv"], weights[p + "bv"])
        save(q), save(k), save(v)
        s = q.shape[0]
        attn = sdpa_dense(q.view(s, hh, dh), k.view(s, hh, dh), v.view(s, hh, dh))
        attn = attn.reshape(s, hh * dh)
        save(attn)
        proj = dense_linear(attn, weights[p + "wo"], weights[p + "bo"])
        seq = dense_add(seq, proj)
        save(seq)
        normed2 = dense_layer_norm(seq, 1, eps=config.eps)
        save(normed2)
        hidden = dense_linear(normed2, weights[p + "w1"], weights[p + "b1"])
        save(hidden)
        mlp = dense_linear(hidden, weights[p + "w2"], weights[p + "b2"])
        seq = dense_add(seq, mlp)
    return seq


# ---------------------------------------------------------------------------
# registrations (domainpar/ops.py:674-696)


def _add_handler(a, b):
    return sharded_elementwise("add", a, b)


def _mul_handler(a, b):
    return sharded_elementwise("mul", a, b)


def _scale_handler(a, s):
    return sharded_elementwise("scale", a, s)


register_handler("aten_like", "add", _add_handler)
register_handler("aten_like", "mul", _mul_handler)
register_handler("aten_like", "scale", _scale_handler)
register_handler("aten_like", "linear", sharded_linear)
register_handler("aten_like", "softmax", sharded_softmax)
register_handler("aten_like", "layer_norm", sharded_layer_norm)
register_dense_reference("add", dense_add)
register_dense_reference("mul", dense_mul)
register_dense_reference("scale", dense_scale)
register_dense_reference("matmul", dense_matmul)
register_dense_reference("linear", dense_linear)
register_dense_reference("softmax", dense_softmax)
register_dense_reference("layer_norm", dense_layer_norm)
