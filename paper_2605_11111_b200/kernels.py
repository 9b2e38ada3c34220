"""Tensor-level wrappers over the C ABI (include/dp_b200.h).

Each wrapper checks devices/dtypes, reads shapes and element strides off the
torch tensors (torch only supplies device memory and the current stream),
and calls exactly one C entry point.  Host (CPU) tensors are rejected: the
domain-parallel kernels have no CPU implementation.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from ._lib import ALGO_AUTO, AttnGeom, ConvGeom, i64_array
from .errors import UnsupportedConfigError

_DT = {torch.float32: _lib.DP_F32, torch.float64: _lib.DP_F64, torch.bfloat16: _lib.DP_BF16}

# algorithm override for tests/benchmarks: "auto" | "simt" | "tc" | "strict"
# (strict = tensor cores for bf16/fp32 or an UnsupportedConfigError, CUDA
# cores only for fp64; auto counts every CUDA-core call in simt_count())
_ALGO_NAMES = {"auto": _lib.ALGO_AUTO, "simt": _lib.ALGO_SIMT, "tc": _lib.ALGO_TC,
               "strict": _lib.ALGO_STRICT}
_algo = ALGO_AUTO


def set_algo(name: str) -> str:
    """Select the conv/attention algorithm globally; returns the previous name."""
    global _algo
    prev = next(k for k, v in _ALGO_NAMES.items() if v == _algo)
    _algo = _ALGO_NAMES[name]
    return prev


def simt_count() -> int:
    """Conv / attention calls routed to the CUDA-core kernels so far in this
    process (fp64, or geometries outside the tcgen05 envelope)."""
    return _lib.simt_count()


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise UnsupportedConfigError(
            f"dtype {t.dtype} unsupported; use float32, float64 or bfloat16") from None


def state_dtype(dtype: torch.dtype) -> torch.dtype:
    """Accumulator dtype of the attention state / conv weight gradient:
    fp64 for fp32/fp64 inputs (the reference's fp64 softmax state,
    domainpar/ops.py:199-214), fp32 for bf16."""
    return torch.float32 if dtype == torch.bfloat16 else torch.float64


def wgrad_dtype(dtype: torch.dtype) -> torch.dtype:
    return torch.float64 if dtype == torch.float64 else torch.float32


def require_device(what: str, *tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise UnsupportedConfigError(
                f"{what}: tensors must be CUDA device tensors (the B200 path has no CPU "
                f"implementation)")
    _lib.load()


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() else 0)


# ---------------------------------------------------------------------------
# data movement


def copy_strided(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[...] = src[...] for same-shape (possibly strided) device tensors:
    the halo face pack/unpack and varlen redistribute kernel."""
    if tuple(dst.shape) != tuple(src.shape) or dst.dtype != src.dtype:
        raise UnsupportedConfigError(
            f"copy_strided: {tuple(src.shape)} {src.dtype} -> {tuple(dst.shape)} {dst.dtype}")
    require_device("copy_strided", dst, src)
    if dst.numel() == 0:
        return
    nd = max(1, dst.dim())
    shape = list(dst.shape) or [1]
    ds = list(dst.stride()) or [1]
    ss = list(src.stride()) or [1]
    rc = _lib.load().dp_copy_strided(nd, i64_array(shape), _ptr(dst), i64_array(ds), _ptr(src),
                                     i64_array(ss), dst.element_size(), _stream(dst))
    _lib.check(rc, "dp_copy_strided")


def accumulate(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst += src (the reverse-halo gradient accumulate)."""
    if tuple(dst.shape) != tuple(src.shape) or dst.dtype != src.dtype:
        raise UnsupportedConfigError("accumulate: shape/dtype mismatch")
    require_device("accumulate", dst, src)
    if dst.numel() == 0:
        return
    nd = max(1, dst.dim())
    rc = _lib.load().dp_accumulate_strided(
        nd, i64_array(list(dst.shape) or [1]), _ptr(dst), i64_array(list(dst.stride()) or [1]),
        _ptr(src), i64_array(list(src.stride()) or [1]), dtype_code(dst), _stream(dst))
    _lib.check(rc, "dp_accumulate_strided")


def convert(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[...] = src[...] converted to dst's dtype (fp32 / fp64 / bf16)."""
    if tuple(dst.shape) != tuple(src.shape):
        raise UnsupportedConfigError(f"convert: {tuple(src.shape)} -> {tuple(dst.shape)}")
    require_device("convert", dst, src)
    if dst.numel() == 0:
        return
    nd = max(1, dst.dim())
    rc = _lib.load().dp_convert_strided(
        nd, i64_array(list(dst.shape) or [1]), _ptr(dst), i64_array(list(dst.stride()) or [1]),
        dtype_code(dst), _ptr(src), i64_array(list(src.stride()) or [1]), dtype_code(src),
        _stream(dst))
    _lib.check(rc, "dp_convert_strided")


def max_into(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst = max(dst, src) elementwise (all_reduce "max" fold)."""
    if tuple(dst.shape) != tuple(src.shape) or dst.dtype != src.dtype:
        raise UnsupportedConfigError("max_into: shape/dtype mismatch")
    require_device("max_into", dst, src)
    if dst.numel() == 0:
        return
    nd = max(1, dst.dim())
    rc = _lib.load().dp_max_strided(
        nd, i64_array(list(dst.shape) or [1]), _ptr(dst), i64_array(list(dst.stride()) or [1]),
        _ptr(src), i64_array(list(src.stride()) or [1]), dtype_code(dst), _stream(dst))
    _lib.check(rc, "dp_max_strided")


def is_dense(t: torch.Tensor) -> bool:
    """Non-overlapping and dense: the elements fill [0, numel) of memory in
    some dim order (any permutation of a contiguous layout)."""
    dims = sorted((s, n) for s, n in zip(t.stride(), t.shape) if n != 1)
    expect = 1
    for s, n in dims:
        if s != expect:
            return False
        expect *= n
    return True


def fill(t: torch.Tensor, value: float) -> torch.Tensor:
    """t[...] = value for a dense device tensor (dp_fill); returns t."""
    require_device("fill", t)
    if t.numel() == 0:
        return t
    if not is_dense(t):
        raise UnsupportedConfigError("fill: tensor must be dense")
    rc = _lib.load().dp_fill(t.numel(), _ptr(t), dtype_code(t), float(value), _stream(t))
    _lib.check(rc, "dp_fill")
    return t


def zeros(shape, dtype, device) -> torch.Tensor:
    """A zero-filled device tensor made by the library (no eager torch kernel)."""
    return fill(torch.empty(tuple(shape), dtype=dtype, device=device), 0.0)


# ---------------------------------------------------------------------------
# convolution


def _pad5(vals, fill=0):
    vals = list(vals)
    return vals + [fill] * (5 - len(vals))


def conv_geom(x: torch.Tensor, x_halo, y_shape, y_strides, c_out: int, kernel, stride, base,
              shard: int, halo_rows: int, out_org=None) -> ConvGeom:
    """Build dp_conv_geom for batched x [B, C, *sp] (main block), optional
    halo block (same dims, `halo_rows` on spatial dim `shard`), output
    shape/strides [B, C_out, *out].  out_org: global index of the produced
    tensor's element 0 per spatial dim (fwd: y, dgrad: dx)."""
    nsp = x.dim() - 2
    if not 1 <= nsp <= 3:
        raise UnsupportedConfigError(f"conv supports 1-3 spatial dims, got {nsp}")
    g = ConvGeom()
    g.nsp = nsp
    g.shard = shard
    g.batch = x.shape[0]
    g.c_in = x.shape[1]
    g.c_out = c_out
    for i in range(3):
        g.in_ext[i] = x.shape[2 + i] if i < nsp else 1
        g.out_ext[i] = y_shape[2 + i] if i < nsp else 1
        g.kernel[i] = kernel[i] if i < nsp else 1
        g.stride[i] = stride[i] if i < nsp else 1
        g.base[i] = base[i] if i < nsp else 0
    g.halo = halo_rows
    for i, v in enumerate(_pad5(x.stride())):
        g.xs[i] = v
    hs = x_halo.stride() if (x_halo is not None and halo_rows) else x.stride()
    for i, v in enumerate(_pad5(hs)):
        g.hs[i] = v
    for i, v in enumerate(_pad5(y_strides)):
        g.ys[i] = v
    for i, v in enumerate(out_org or ()):
        g.out_org[i] = int(v)
    return g


def _workspace(g, code, which, device):
    nbytes = _lib.load().dp_conv_workspace(ctypes.byref(g), code, _algo, which)
    if nbytes < 0:
        _lib.check(_lib.DP_ERR_UNSUPPORTED, "dp_conv_workspace")
    ws = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)
    return ws, int(ws.numel())


def conv_fwd(x, x_halo, w, y, *, kernel, stride, base, shard, halo_rows, out_org=None) -> None:
    require_device("conv_fwd", x, x_halo, w, y)
    g = conv_geom(x, x_halo, y.shape, y.stride(), w.shape[0], kernel, stride, base, shard,
                  halo_rows, out_org)
    code = dtype_code(x)
    ws, nb = _workspace(g, code, _lib.CONV_FWD, x.device)
    rc = _lib.load().dp_conv_fwd(ctypes.byref(g), code, _algo, _ptr(x), _ptr(x_halo), _ptr(w),
                                 _ptr(y), _ptr(ws), nb, _stream(x))
    _lib.check(rc, "dp_conv_fwd")


def conv_dgrad(dy, w, dx, dx_halo, *, kernel, stride, base, shard, halo_rows,
               out_org=None) -> None:
    require_device("conv_dgrad", dy, w, dx, dx_halo)
    g = conv_geom(dx, dx_halo, dy.shape, dy.stride(), w.shape[0], kernel, stride, base, shard,
                  halo_rows, out_org)
    code = dtype_code(dy)
    ws, nb = _workspace(g, code, _lib.CONV_DGRAD, dy.device)
    rc = _lib.load().dp_conv_dgrad(ctypes.byref(g), code, _algo, _ptr(dy), _ptr(w), _ptr(dx),
                                   _ptr(dx_halo), _ptr(ws), nb, _stream(dy))
    _lib.check(rc, "dp_conv_dgrad")


def conv_wgrad(x, x_halo, dy, dw, *, kernel, stride, base, shard, halo_rows) -> None:
    """dw (contiguous, wgrad_dtype) = this rank's weight-gradient partial."""
    require_device("conv_wgrad", x, x_halo, dy, dw)
    g = conv_geom(x, x_halo, dy.shape, dy.stride(), dw.shape[0], kernel, stride, base, shard,
                  halo_rows)
    code = dtype_code(x)
    ws, nb = _workspace(g, code, _lib.CONV_WGRAD, x.device)
    rc = _lib.load().dp_conv_wgrad(ctypes.byref(g), code, _algo, _ptr(x), _ptr(x_halo),
                                   _ptr(dy), _ptr(dw), _ptr(ws), nb, _stream(x))
    _lib.check(rc, "dp_conv_wgrad")


# ---------------------------------------------------------------------------
# fp32 conv with operands split once (bf16x3, include/dp_b200.h dp_conv_x3_*)

X3_X, X3_XHALO, X3_DY = 0, 1, 2


def x3_active(x, x_halo, y_shape, y_strides, c_out, *, kernel, stride, base, shard,
              halo_rows) -> bool:
    """True when fp32 convs of this geometry (fwd, dgrad AND wgrad) run on the
    tensor cores as bf16x3 — then the caller splits x / dy once and uses the
    *_parts entry points (the CUDA-core algorithm has no split form)."""
    if x.dtype != torch.float32 or _algo == _lib.ALGO_SIMT:
        return False
    g = conv_geom(x, x_halo, y_shape, y_strides, c_out, kernel, stride, base, shard, halo_rows)
    lib = _lib.load()
    return all(lib.dp_conv_x3_parts_workspace(ctypes.byref(g), w) >= 0
               for w in (_lib.CONV_FWD, _lib.CONV_DGRAD, _lib.CONV_WGRAD))


def x3_split(t, operand, g) -> torch.Tensor:
    """The 3 bf16 parts of fp32 operand `t` ([3][B][s0][s1][C] bf16) for geometry g."""
    require_device("x3_split", t)
    lib = _lib.load()
    nbytes = lib.dp_conv_x3_operand_bytes(ctypes.byref(g), operand)
    if nbytes < 0:
        _lib.check(_lib.DP_ERR_UNSUPPORTED, "dp_conv_x3_operand_bytes")
    parts = torch.empty(max(int(nbytes) // 2, 1), dtype=torch.bfloat16, device=t.device)
    if nbytes:
        _lib.check(lib.dp_conv_x3_split(ctypes.byref(g), operand, _ptr(t), _ptr(parts),
                                        _stream(t)), "dp_conv_x3_split")
    return parts


def _x3_ws(g, which, device):
    nbytes = _lib.load().dp_conv_x3_parts_workspace(ctypes.byref(g), which)
    if nbytes < 0:
        _lib.check(_lib.DP_ERR_UNSUPPORTED, "dp_conv_x3_parts_workspace")
    ws = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)
    return ws, int(ws.numel())


def conv_fwd_x3(x, x_halo, xp, xhp, w, y, *, kernel, stride, base, shard, halo_rows,
                out_org=None) -> None:
    """conv_fwd of fp32 x whose parts xp (and halo parts xhp) are already split."""
    require_device("conv_fwd_x3", xp, w, y)
    g = conv_geom(x, x_halo, y.shape, y.stride(), w.shape[0], kernel, stride, base, shard,
                  halo_rows, out_org)
    ws, nb = _x3_ws(g, _lib.CONV_FWD, y.device)
    _lib.check(_lib.load().dp_conv_x3_fwd_parts(ctypes.byref(g), _ptr(xp), _ptr(xhp), _ptr(w),
                                                _ptr(y), _ptr(ws), nb, _stream(y)),
               "dp_conv_x3_fwd_parts")


def conv_dgrad_x3(dy, dyp, w, dx, dx_halo, *, kernel, stride, base, shard, halo_rows,
                  out_org=None) -> None:
    require_device("conv_dgrad_x3", dyp, w, dx, dx_halo)
    g = conv_geom(dx, dx_halo, dy.shape, dy.stride(), w.shape[0], kernel, stride, base, shard,
                  halo_rows, out_org)
    ws, nb = _x3_ws(g, _lib.CONV_DGRAD, dx.device)
    _lib.check(_lib.load().dp_conv_x3_dgrad_parts(ctypes.byref(g), _ptr(dyp), _ptr(w), _ptr(dx),
                                                  _ptr(dx_halo), _ptr(ws), nb, _stream(dx)),
               "dp_conv_x3_dgrad_parts")


def conv_wgrad_x3(x, x_halo, xp, xhp, dy, dyp, dw, *, kernel, stride, base, shard,
                  halo_rows) -> None:
    require_device("conv_wgrad_x3", xp, dyp, dw)
    g = conv_geom(x, x_halo, dy.shape, dy.stride(), dw.shape[0], kernel, stride, base, shard,
                  halo_rows)
    ws, nb = _x3_ws(g, _lib.CONV_WGRAD, dw.device)
    _lib.check(_lib.load().dp_conv_x3_wgrad_parts(ctypes.byref(g), _ptr(xp), _ptr(xhp), _ptr(dyp),
                                                  _ptr(dw), _ptr(ws), nb, _stream(dw)),
               "dp_conv_x3_wgrad_parts")


# ---------------------------------------------------------------------------
# attention


def _as3(t: torch.Tensor) -> torch.Tensor:
    """[S, d] -> [S, 1, d]; [S, H, d] stays."""
    return t.unsqueeze(1) if t.dim() == 2 else t


def attn_geom(q3, k3, v3, o3, scale) -> AttnGeom:
    g = AttnGeom()
    g.sq, g.heads, g.dim = q3.shape
    g.sk = k3.shape[0]
    g.q_rs, g.q_hs = q3.stride(0), q3.stride(1)
    g.k_rs, g.k_hs = k3.stride(0), k3.stride(1)
    g.v_rs, g.v_hs = v3.stride(0), v3.stride(1)
    o = o3 if o3 is not None else q3
    g.o_rs, g.o_hs = o.stride(0), o.stride(1)
    g.scale = float(scale)
    for t in (q3, k3, v3, o3):
        if t is not None and t.numel() and t.stride(2) != 1:
            raise UnsupportedConfigError("attention: head dim must be unit-stride")
    return g


def attn_fwd_update(q, k, v, m, l, acc, scale) -> None:
    require_device("attn_fwd_update", q, k, v, m, l, acc)
    q3, k3, v3 = _as3(q), _as3(k), _as3(v)
    g = attn_geom(q3, k3, v3, None, scale)
    rc = _lib.load().dp_attn_fwd_update(ctypes.byref(g), dtype_code(q), _algo, _ptr(q3),
                                        _ptr(k3), _ptr(v3), _ptr(m), _ptr(l), _ptr(acc),
                                        _stream(q))
    _lib.check(rc, "dp_attn_fwd_update")


def attn_finalize(q, m, l, acc, out, lse, scale) -> None:
    require_device("attn_finalize", m, l, acc, out, lse)
    q3, o3 = _as3(q), _as3(out)
    g = attn_geom(q3, q3, q3, o3, scale)
    rc = _lib.load().dp_attn_finalize(ctypes.byref(g), dtype_code(out), _ptr(m), _ptr(l),
                                      _ptr(acc), _ptr(o3), _ptr(lse), _stream(out))
    _lib.check(rc, "dp_attn_finalize")


def attn_bwd_preprocess(o, do, delta) -> None:
    require_device("attn_bwd_preprocess", o, do, delta)
    o3, d3 = _as3(o), _as3(do)
    if o3.stride() != d3.stride():
        d3 = d3.contiguous()
        o3 = o3.contiguous()
    g = attn_geom(o3, o3, o3, o3, 1.0)
    rc = _lib.load().dp_attn_bwd_preprocess(ctypes.byref(g), dtype_code(o), _ptr(o3), _ptr(d3),
                                            _ptr(delta), _stream(o))
    _lib.check(rc, "dp_attn_bwd_preprocess")


def attn_bwd_update(q, k, v, do, lse, delta, dq, dk, dv, scale) -> None:
    require_device("attn_bwd_update", q, k, v, do, lse, delta, dq, dk, dv)
    q3, k3, v3, d3 = _as3(q), _as3(k), _as3(v), _as3(do)
    g = attn_geom(q3, k3, v3, d3, scale)
    rc = _lib.load().dp_attn_bwd_update(ctypes.byref(g), dtype_code(q), _algo, _ptr(q3),
                                        _ptr(k3), _ptr(v3), _ptr(d3), _ptr(lse), _ptr(delta),
                                        _ptr(dq), _ptr(dk), _ptr(dv), _stream(q))
    _lib.check(rc, "dp_attn_bwd_update")


def default_scale(d: int) -> float:
    """1/sqrt(d) as a Python float (domainpar/ops.py:268)."""
    return 1.0 / math.sqrt(d)


# ---------------------------------------------------------------------------
# normalisations and pointwise ops


def contiguous(t: torch.Tensor) -> torch.Tensor:
    """`t` itself when contiguous, else a contiguous copy made by dp_copy_strided."""
    if t.is_contiguous():
        return t
    out = torch.empty(t.shape, dtype=t.dtype, device=t.device)
    copy_strided(out, t)
    return out


def _view3(shape, dim):
    outer = math.prod(shape[:dim])
    inner = math.prod(shape[dim + 1:])
    return outer, shape[dim], inner


def norm_stats(kind: int, x: torch.Tensor, dim: int, aux=None) -> torch.Tensor:
    """fp64 statistics of contiguous `x` reduced over `dim` (dp_norm_stats):
    [2, cells] moments (kind 0), [1, cells] max (1) or exp-sum (2)."""
    require_device("norm_stats", x, aux)
    outer, n, inner = _view3(list(x.shape), dim)
    nstat = 2 if kind == _lib.NORM_MOMENTS else 1
    stats = torch.empty((nstat, outer * inner), dtype=torch.float64, device=x.device)
    lib = _lib.load()
    nb = int(lib.dp_norm_workspace(kind, outer, n, inner))
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=x.device)
    rc = lib.dp_norm_stats(kind, outer, n, inner, _ptr(x), i64_array([n * inner, inner, 1]),
                           dtype_code(x), _ptr(aux), _ptr(stats), _ptr(ws), ws.numel(),
                           _stream(x))
    _lib.check(rc, "dp_norm_stats")
    return stats


def norm_apply(kind: int, x: torch.Tensor, dim: int, stats: torch.Tensor, aux, count: float,
               eps: float = 0.0) -> torch.Tensor:
    """Normalised copy of contiguous `x` from GLOBAL statistics (dp_norm_apply)."""
    require_device("norm_apply", x, stats, aux)
    outer, n, inner = _view3(list(x.shape), dim)
    y = torch.empty(x.shape, dtype=x.dtype, device=x.device)
    st = i64_array([n * inner, inner, 1])
    rc = _lib.load().dp_norm_apply(kind, outer, n, inner, _ptr(x), st, _ptr(y), st,
                                   dtype_code(x), _ptr(stats), _ptr(aux), float(count),
                                   float(eps), _stream(x))
    _lib.check(rc, "dp_norm_apply")
    return y


def elementwise(op: int, a: torch.Tensor, b=None, scalar: float = 0.0) -> torch.Tensor:
    """out = a (+|*) b, or a * scalar (dp_elementwise); contiguous result."""
    require_device("elementwise", a, b if isinstance(b, torch.Tensor) else None)
    a = contiguous(a)
    if isinstance(b, torch.Tensor):
        b = contiguous(b.to(a.dtype))
    out = torch.empty(a.shape, dtype=a.dtype, device=a.device)
    rc = _lib.load().dp_elementwise(op, a.numel(), _ptr(a),
                                    _ptr(b) if isinstance(b, torch.Tensor) else None,
                                    float(scalar), _ptr(out), dtype_code(a), _stream(a))
    _lib.check(rc, "dp_elementwise")
    return out
