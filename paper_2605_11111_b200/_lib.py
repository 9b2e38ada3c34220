"""ctypes binding of the in-tree C-ABI library `libdpb200.so` (include/dp_b200.h).

The library is built by `__graft_entry__.build()` (nvcc, sm_100a) and loaded
from this package directory — never from site-packages or a JIT cache — so
the round-end evidence of which native code ran points at this file.  A
missing library is a hard error for every device op: there is no CPU path.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CollectiveError, DeviceError, UnsupportedConfigError

LIB_NAME = "libdpb200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

DP_OK, DP_ERR_INVALID, DP_ERR_UNSUPPORTED, DP_ERR_CUDA, DP_ERR_COMM, DP_ERR_TIMEOUT = \
    0, 1, 2, 3, 4, 5
REDUCE_SUM, REDUCE_MAX = 0, 1
NCCL_UNIQUE_ID_BYTES = 128
DP_F32, DP_F64, DP_BF16 = 0, 1, 2
ALGO_AUTO, ALGO_SIMT, ALGO_TC, ALGO_STRICT = 0, 1, 2, 3
CONV_FWD, CONV_DGRAD, CONV_WGRAD = 0, 1, 2
NORM_MOMENTS, NORM_MAX, NORM_EXPSUM = 0, 1, 2
EW_ADD, EW_MUL, EW_SCALE = 0, 1, 2

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int)
_vpp = ctypes.POINTER(ctypes.c_void_p)


class ConvGeom(ctypes.Structure):
    """Mirror of `dp_conv_geom` (include/dp_b200.h)."""

    _fields_ = [
        ("nsp", _i32), ("shard", _i32),
        ("batch", _i64), ("c_in", _i64), ("c_out", _i64),
        ("in_ext", _i64 * 3), ("halo", _i64), ("out_ext", _i64 * 3),
        ("kernel", _i32 * 3), ("stride", _i32 * 3), ("base", _i64 * 3),
        ("xs", _i64 * 5), ("hs", _i64 * 5), ("ys", _i64 * 5), ("out_org", _i64 * 3),
    ]


class AttnGeom(ctypes.Structure):
    """Mirror of `dp_attn_geom` (include/dp_b200.h)."""

    _fields_ = [
        ("sq", _i64), ("sk", _i64), ("heads", _i64), ("dim", _i64),
        ("q_rs", _i64), ("q_hs", _i64), ("k_rs", _i64), ("k_hs", _i64),
        ("v_rs", _i64), ("v_hs", _i64), ("o_rs", _i64), ("o_hs", _i64),
        ("scale", ctypes.c_double),
    ]


# name -> (restype, argtypes); every symbol include/dp_b200.h declares
SIGNATURES = {
    "dp_abi_version": (ctypes.c_int, []),
    "dp_last_error": (ctypes.c_char_p, []),
    "dp_launch_count": (ctypes.c_uint64, []),
    "dp_simt_count": (ctypes.c_uint64, []),
    "dp_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)] * 3),
    "dp_copy_strided": (ctypes.c_int, [ctypes.c_int, _i64p, _vp, _i64p, _vp, _i64p,
                                       ctypes.c_int, _vp]),
    "dp_accumulate_strided": (ctypes.c_int, [ctypes.c_int, _i64p, _vp, _i64p, _vp, _i64p,
                                             ctypes.c_int, _vp]),
    "dp_convert_strided": (ctypes.c_int, [ctypes.c_int, _i64p, _vp, _i64p, ctypes.c_int, _vp,
                                          _i64p, ctypes.c_int, _vp]),
    "dp_max_strided": (ctypes.c_int, [ctypes.c_int, _i64p, _vp, _i64p, _vp, _i64p, ctypes.c_int,
                                      _vp]),
    "dp_fill": (ctypes.c_int, [ctypes.c_int64, _vp, ctypes.c_int, ctypes.c_double, _vp]),
    "dp_conv_workspace": (ctypes.c_int64, [ctypes.POINTER(ConvGeom), ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int]),
    "dp_conv_fwd": (ctypes.c_int, [ctypes.POINTER(ConvGeom), ctypes.c_int, ctypes.c_int,
                                   _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]),
    "dp_conv_dgrad": (ctypes.c_int, [ctypes.POINTER(ConvGeom), ctypes.c_int, ctypes.c_int,
                                     _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]),
    "dp_conv_wgrad": (ctypes.c_int, [ctypes.POINTER(ConvGeom), ctypes.c_int, ctypes.c_int,
                                     _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]),
    "dp_conv_x3_operand_bytes": (ctypes.c_int64, [ctypes.POINTER(ConvGeom), ctypes.c_int]),
    "dp_conv_x3_split": (ctypes.c_int, [ctypes.POINTER(ConvGeom), ctypes.c_int, _vp, _vp, _vp]),
    "dp_conv_x3_parts_workspace": (ctypes.c_int64, [ctypes.POINTER(ConvGeom), ctypes.c_int]),
    "dp_conv_x3_fwd_parts": (ctypes.c_int, [ctypes.POINTER(ConvGeom), _vp, _vp, _vp, _vp, _vp,
                                            ctypes.c_int64, _vp]),
    "dp_conv_x3_dgrad_parts": (ctypes.c_int, [ctypes.POINTER(ConvGeom), _vp, _vp, _vp, _vp, _vp,
                                              ctypes.c_int64, _vp]),
    "dp_conv_x3_wgrad_parts": (ctypes.c_int, [ctypes.POINTER(ConvGeom), _vp, _vp, _vp, _vp, _vp,
                                              ctypes.c_int64, _vp]),
    "dp_attn_fwd_update": (ctypes.c_int, [ctypes.POINTER(AttnGeom), ctypes.c_int, ctypes.c_int,
                                          _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dp_attn_finalize": (ctypes.c_int, [ctypes.POINTER(AttnGeom), ctypes.c_int,
                                        _vp, _vp, _vp, _vp, _vp, _vp]),
    "dp_attn_bwd_preprocess": (ctypes.c_int, [ctypes.POINTER(AttnGeom), ctypes.c_int,
                                              _vp, _vp, _vp, _vp]),
    "dp_attn_bwd_update": (ctypes.c_int, [ctypes.POINTER(AttnGeom), ctypes.c_int, ctypes.c_int,
                                          _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dp_norm_workspace": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64]),
    "dp_norm_stats": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     _vp, _i64p, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int64,
                                     _vp]),
    "dp_norm_apply": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     _vp, _i64p, _vp, _i64p, ctypes.c_int, _vp, _vp,
                                     ctypes.c_double, ctypes.c_double, _vp]),
    "dp_elementwise": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, _vp, _vp, ctypes.c_double,
                                      _vp, ctypes.c_int, _vp]),
    # communicators / exchanges (comm.cu)
    "dp_comm_load": (ctypes.c_int, [ctypes.c_char_p]),
    "dp_comm_version": (ctypes.c_int, [_i32p]),
    "dp_comm_unique_id": (ctypes.c_int, [_vp]),
    "dp_comm_init": (ctypes.c_int, [_vpp, ctypes.c_int, ctypes.c_int, _vp]),
    "dp_comm_split": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vpp]),
    "dp_comm_info": (ctypes.c_int, [_vp, _i32p, _i32p]),
    "dp_comm_destroy": (ctypes.c_int, [_vp]),
    "dp_comm_abort": (ctypes.c_int, [_vp]),
    "dp_comm_exchange": (ctypes.c_int, [_vp, ctypes.c_int, _i32p, _i32p, _vpp, _i64p, _vp]),
    "dp_halo_sendrecv": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int64, _vp,
                                        ctypes.c_int64, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                        _vp]),
    "dp_ring_step": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp]),
    "dp_varlen_allgather": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, _i64p, _i64p, _vp]),
    "dp_varlen_alltoall": (ctypes.c_int, [_vp, _vpp, _i64p, _vpp, _i64p, _vp]),
    "dp_allreduce": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    _vp]),
    "dp_comm_wait": (ctypes.c_int, [_vp, _vp, ctypes.c_double]),
}

_LIB = None


def load():
    """Load (once) and return the library; DeviceError when it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_NAME} is not built ({LIB_PATH}); run `python -c \"import __graft_entry__ as g; "
            f"g.build()\"` — the domain-parallel ops have no CPU implementation")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.dp_abi_version() != 1:
        raise DeviceError(f"{LIB_NAME} ABI version {lib.dp_abi_version()} != 1")
    _LIB = lib
    return lib


def available() -> bool:
    try:
        load()
        return True
    except (DeviceError, OSError):
        return False


def check(rc: int, what: str) -> None:
    """Map a DP_ERR_* code to the package's error types (NCCL failures and
    watchdog timeouts are CollectiveErrors, as the reference's queue
    timeouts, domainpar/mesh.py:196-206)."""
    if rc == DP_OK:
        return
    msg = load().dp_last_error().decode(errors="replace")
    if rc == DP_ERR_UNSUPPORTED:
        raise UnsupportedConfigError(f"{what}: {msg}")
    if rc in (DP_ERR_COMM, DP_ERR_TIMEOUT):
        raise CollectiveError(f"{what}: {msg}")
    raise DeviceError(f"{what} failed (code {rc}): {msg}")


def launch_count() -> int:
    return int(load().dp_launch_count())


def simt_count() -> int:
    """Conv / attention calls the library routed to its CUDA-core kernels."""
    return int(load().dp_simt_count())


def i64_array(values):
    values = [int(v) for v in values]
    return (ctypes.c_int64 * max(1, len(values)))(*values)
