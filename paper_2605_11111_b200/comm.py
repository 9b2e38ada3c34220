"""NCCL communicators through the library's C ABI (include/dp_b200.h,
csrc/comm.cu): the data plane of the one-process-per-GPU mesh.

torch.distributed (gloo) is only the control plane here — rendezvous, the
unique-id broadcast, host metadata and barriers.  Every device byte that
crosses a GPU boundary goes through `dp_comm_exchange` / `dp_allreduce`,
enqueued on the caller's CUDA stream.  Replaces the reference's per-pair
queues (domainpar/mesh.py:252-403).
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .errors import CollectiveError

_LOADED = False


def _nccl_path() -> str | None:
    """The libnccl.so.2 torch ships (already mapped into this process when
    torch's CUDA side is loaded); None lets the loader search."""
    try:
        import nvidia.nccl as n

        for base in list(n.__path__):
            p = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except Exception:  # noqa: BLE001 - fall back to the loader's search path
        pass
    return None


def load() -> None:
    """Resolve NCCL inside libdpb200.so (once)."""
    global _LOADED
    if _LOADED:
        return
    lib = _lib.load()
    path = _nccl_path()
    _lib.check(lib.dp_comm_load(path.encode() if path else None), "dp_comm_load")
    _LOADED = True


def version() -> int:
    load()
    v = ctypes.c_int(0)
    _lib.check(_lib.load().dp_comm_version(ctypes.byref(v)), "dp_comm_version")
    return int(v.value)


def unique_id() -> bytes:
    load()
    buf = ctypes.create_string_buffer(_lib.NCCL_UNIQUE_ID_BYTES)
    _lib.check(_lib.load().dp_comm_unique_id(buf), "dp_comm_unique_id")
    return buf.raw


def _stream_ptr(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr() if t.numel() else 0


class NcclComm:
    """One NCCL communicator (a mesh-axis line, or the world)."""

    def __init__(self, handle: ctypes.c_void_p, rank: int, size: int):
        self.handle = handle
        self.rank = rank
        self.size = size

    @classmethod
    def init(cls, world: int, rank: int, uid: bytes) -> "NcclComm":
        """Collective over `world` ranks on the current CUDA device."""
        load()
        if len(uid) != _lib.NCCL_UNIQUE_ID_BYTES:
            raise CollectiveError(f"NCCL unique id must be {_lib.NCCL_UNIQUE_ID_BYTES} bytes")
        h = ctypes.c_void_p()
        _lib.check(_lib.load().dp_comm_init(ctypes.byref(h), world, rank,
                                            ctypes.create_string_buffer(uid, len(uid))),
                   "dp_comm_init")
        return cls(h, rank, world)

    def split(self, color: int, key: int) -> "NcclComm | None":
        """Collective over this communicator (ncclCommSplit)."""
        h = ctypes.c_void_p()
        _lib.check(_lib.load().dp_comm_split(self.handle, color, key, ctypes.byref(h)),
                   "dp_comm_split")
        if not h.value:
            return None
        r, n = ctypes.c_int(0), ctypes.c_int(0)
        _lib.check(_lib.load().dp_comm_info(h, ctypes.byref(r), ctypes.byref(n)), "dp_comm_info")
        return NcclComm(h, int(r.value), int(n.value))

    def exchange(self, ops, stream=None) -> None:
        """ops = [(peer, is_recv, tensor)]: one grouped NCCL round of dense
        device buffers, sent / received as bytes in memory order."""
        n = len(ops)
        if n == 0:
            return
        peers = (ctypes.c_int * n)(*[int(p) for p, _, _ in ops])
        kinds = (ctypes.c_int * n)(*[1 if r else 0 for _, r, _ in ops])
        bufs = (ctypes.c_void_p * n)(*[_ptr(t) for _, _, t in ops])
        nbytes = (ctypes.c_int64 * n)(*[t.numel() * t.element_size() for _, _, t in ops])
        _lib.check(_lib.load().dp_comm_exchange(self.handle, n, peers, kinds, bufs, nbytes,
                                                _stream_ptr(stream)), "dp_comm_exchange")

    def ring_step(self, send: torch.Tensor, recv: torch.Tensor, stream=None) -> None:
        _lib.check(_lib.load().dp_ring_step(
            self.handle, _ptr(send), send.numel() * send.element_size(), _ptr(recv),
            recv.numel() * recv.element_size(), _stream_ptr(stream)), "dp_ring_step")

    def halo_sendrecv(self, left: int, right: int, send_left, send_right, recv_left, recv_right,
                      stream=None) -> None:
        def pb(t):
            return (_ptr(t), t.numel() * t.element_size()) if t is not None else (0, 0)

        sl, sr, rl, rr = pb(send_left), pb(send_right), pb(recv_left), pb(recv_right)
        _lib.check(_lib.load().dp_halo_sendrecv(self.handle, left, right, sl[0], sl[1], sr[0],
                                                sr[1], rl[0], rl[1], rr[0], rr[1],
                                                _stream_ptr(stream)), "dp_halo_sendrecv")

    def allreduce(self, send: torch.Tensor, recv: torch.Tensor, op: str = "sum",
                  stream=None) -> None:
        from .kernels import dtype_code

        rop = _lib.REDUCE_SUM if op == "sum" else _lib.REDUCE_MAX
        _lib.check(_lib.load().dp_allreduce(self.handle, _ptr(send), _ptr(recv), send.numel(),
                                            dtype_code(send), rop, _stream_ptr(stream)),
                   "dp_allreduce")

    def wait(self, stream=None, timeout: float = 0.0) -> None:
        """Watchdog wait: an async NCCL error or the timeout aborts the
        communicator and raises CollectiveError."""
        _lib.check(_lib.load().dp_comm_wait(self.handle, _stream_ptr(stream), float(timeout)),
                   "dp_comm_wait")

    def destroy(self) -> None:
        if self.handle is not None and self.handle.value:
            _lib.check(_lib.load().dp_comm_destroy(self.handle), "dp_comm_destroy")
        self.handle = None

    def abort(self) -> None:
        if self.handle is not None and self.handle.value:
            _lib.load().dp_comm_abort(self.handle)
        self.handle = None
