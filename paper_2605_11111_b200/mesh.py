"""Device mesh, rank contexts, and the collectives of the domain-parallel path.

Reference: domainpar/mesh.py (thread ranks over per-pair queues).  The B200
design keeps the reference's *API* — DeviceMesh, RankContext, AxisGroup,
all_reduce / all_gather_varlen / ring_shift / halo_exchange / barrier,
spawn_mesh — and replaces the runtime underneath with two transports:

  * "nccl"/"gloo": one OS process per GPU (or per CPU rank), torch.distributed
    process groups, one NCCL communicator per mesh-axis line.  This is the
    production path (bench.py under torchrun uses `init_mesh`).
  * "thread": the reference's execution model — one Python thread per rank
    in this process, per-pair FIFO mailboxes — but the payloads are CUDA
    tensors resident on one device.  It lets the full sharded algorithm
    (plans, face packing, exchanges, kernels) run with R ranks on a single
    B200, which is how the GPU parity suite exercises R in {1..8}.

Message sizes on the hot path are computed locally from replicated
metadata (ShardTensor.shard_shapes), so the device path never needs the
reference's width/shape handshakes.  The generic public collectives that
*do* take per-rank sizes (halo_exchange widths, all_gather_varlen extents)
run one small host-side metadata round first, exactly mirroring the
reference's handshake (domainpar/mesh.py:347-355, :292-301).

Collective accounting follows the reference (mesh.py:260,289,308,341,392):
ctx.collective_count grows by exactly one per logical collective call, no
matter how many NCCL calls implement it.
"""

from __future__ import annotations

import os
import queue
import threading
import time
from collections import deque
from dataclasses import dataclass

import torch

from .errors import CollectiveError, DimensionError, HaloError, MeshError

TIMEOUT_ENV = "DP_COLLECTIVE_TIMEOUT_SECS"
DEFAULT_TIMEOUT = 30.0
_POLL = 0.002
REDUCE_OPS = ("sum", "max")

__all__ = [
    "DeviceMesh", "RankContext", "AxisGroup", "all_reduce", "all_gather_varlen",
    "ring_shift", "halo_exchange", "barrier", "spawn_mesh", "init_mesh", "NativeTransport",
    "TIMEOUT_ENV", "REDUCE_OPS",
]


class PeerAbort(CollectiveError):
    """Raised on ranks that stop because some *other* rank failed first; these
    are filtered out of MeshError's primary failures (as the reference's
    _PeerFailure, mesh.py:43-44)."""


# ---------------------------------------------------------------------------
# geometry


@dataclass(frozen=True)
class DeviceMesh:
    """1-D or 2-D grid of ranks with named axes; rank ids are row-major."""

    shape: tuple
    axis_names: tuple

    def __post_init__(self):
        shape = tuple(int(s) for s in self.shape)
        names = tuple(self.axis_names)
        object.__setattr__(self, "shape", shape)
        object.__setattr__(self, "axis_names", names)
        if len(shape) not in (1, 2):
            raise DimensionError(f"mesh must have 1 or 2 axes, got shape {shape}")
        if min(shape) < 1:
            raise DimensionError(f"mesh axis extents must be >= 1, got {shape}")
        if len(names) != len(shape):
            raise DimensionError(f"{len(names)} axis names for {len(shape)} axes")
        if len(set(names)) != len(names):
            raise DimensionError(f"duplicate mesh axis names {names}")

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def world_size(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    def axis_index(self, name: str) -> int:
        if name not in self.axis_names:
            raise DimensionError(f"no mesh axis named {name!r}; have {self.axis_names}")
        return self.axis_names.index(name)

    def coords_of(self, rank_id: int) -> tuple:
        if not 0 <= rank_id < self.world_size:
            raise DimensionError(f"rank {rank_id} out of range for mesh {self.shape}")
        if self.ndim == 1:
            return (rank_id,)
        return (rank_id // self.shape[1], rank_id % self.shape[1])

    def rank_of(self, coords) -> int:
        coords = tuple(int(c) for c in coords)
        if len(coords) != self.ndim:
            raise DimensionError(f"coords {coords} for {self.ndim}-D mesh")
        for c, n in zip(coords, self.shape):
            if not 0 <= c < n:
                raise DimensionError(f"coords {coords} out of mesh {self.shape}")
        if self.ndim == 1:
            return coords[0]
        return coords[0] * self.shape[1] + coords[1]

    def line(self, coords, axis: int) -> tuple:
        """Rank ids along `axis` through `coords`, in coordinate order."""
        c = list(coords)
        out = []
        for i in range(self.shape[axis]):
            c[axis] = i
            out.append(self.rank_of(c))
        return tuple(out)


# ---------------------------------------------------------------------------
# transports


def _resolve_timeout(timeout) -> float:
    if timeout is not None:
        return float(timeout)
    raw = os.environ.get(TIMEOUT_ENV)
    if raw is None:
        return DEFAULT_TIMEOUT
    try:
        return float(raw)
    except ValueError:
        raise DimensionError(f"{TIMEOUT_ENV}={raw!r} is not a number") from None


class _ThreadRuntime:
    """Shared state of one thread-mesh run: n*n mailboxes plus flags."""

    def __init__(self, mesh: DeviceMesh, timeout: float):
        n = mesh.world_size
        self.mesh = mesh
        self.timeout = timeout
        self.box = {(s, d): queue.SimpleQueue() for s in range(n) for d in range(n)}
        self.finished = [threading.Event() for _ in range(n)]
        self.abort = threading.Event()


class _Done:
    def wait(self) -> None:
        return None


class _Pending:
    """Outstanding point-to-point works of one exchange round (buffers kept
    alive until waited; `after` = host->device copies of staged receives)."""

    def __init__(self, works, keep, after=()):
        self.works = works
        self.keep = keep
        self.after = list(after)

    def wait(self) -> None:
        for w in self.works:
            w.wait()
        for dst, host in self.after:
            dst.copy_(host)
        self.works = []
        self.keep = []
        self.after = []


class ThreadTransport:
    """Rank-to-rank FIFO mailboxes inside one process (one device)."""

    kind = "thread"

    def __init__(self, runtime: _ThreadRuntime, rank: int):
        self.rt = runtime
        self.rank = rank

    # -- raw messaging ---------------------------------------------------
    def _put(self, dst: int, payload) -> None:
        self.rt.box[(self.rank, dst)].put(payload)

    def _get(self, src: int):
        rt = self.rt
        box = rt.box[(src, self.rank)]
        deadline = time.monotonic() + rt.timeout
        while True:
            try:
                return box.get(timeout=_POLL)
            except queue.Empty:
                pass
            if rt.abort.is_set():
                raise PeerAbort(f"rank {self.rank}: unwinding, another rank failed")
            if rt.finished[src].is_set() and box.empty():
                raise CollectiveError(f"rank {self.rank}: rank {src} finished without sending")
            if time.monotonic() > deadline:
                raise CollectiveError(
                    f"rank {self.rank}: timed out after {rt.timeout:.3g}s waiting for rank {src}")

    # -- transport API ---------------------------------------------------
    def exchange(self, sends, recvs) -> None:
        """Grouped point-to-point: `sends` = [(dst, tensor)], `recvs` =
        [(src, out)] with `out` preallocated.  Senders hand over the tensor
        object itself; all ranks share the device's stream order, so the
        receiver's copy is ordered after the sender's producer kernels."""
        for dst, t in sends:
            self._put(dst, t)
        for src, out in recvs:
            got = self._get(src)
            if tuple(got.shape) != tuple(out.shape) or got.dtype != out.dtype:
                raise CollectiveError(
                    f"rank {self.rank}: expected {tuple(out.shape)} {out.dtype} from rank "
                    f"{src}, got {tuple(got.shape)} {got.dtype}")
            if got.numel():
                _copy_into(out, got)

    def exchange_start(self, sends, recvs):
        """Thread mailboxes complete eagerly; the handle is already done."""
        self.exchange(sends, recvs)
        return _Done()

    def exchange_any(self, sends, srcs) -> list:
        """Like exchange, but receive whatever tensor each source sent."""
        for dst, t in sends:
            self._put(dst, t)
        return [self._get(s) for s in srcs]

    def gather_meta(self, members, me: int, obj) -> list:
        for i, r in enumerate(members):
            if i != me:
                self._put(r, ("meta", obj))
        out = []
        for i, r in enumerate(members):
            if i == me:
                out.append(obj)
            else:
                tag, val = self._get(r)
                out.append(val)
        return out

    def send_meta(self, dst, obj) -> None:
        self._put(dst, ("meta", obj))

    def recv_meta(self, src):
        return self._get(src)[1]

    def all_reduce(self, members, me: int, t: torch.Tensor, op: str) -> torch.Tensor:
        """Fixed member-order fold on every rank: bitwise identical results
        everywhere, the reference's determinism contract (mesh.py:271-277)."""
        parts = self.exchange_any([(r, t) for i, r in enumerate(members) if i != me],
                                  [r for i, r in enumerate(members) if i != me])
        parts.insert(me, t)
        for i, p in enumerate(parts):
            if tuple(p.shape) != tuple(parts[0].shape) or p.dtype != parts[0].dtype:
                raise CollectiveError(
                    f"all_reduce contribution mismatch: member 0 has {tuple(parts[0].shape)} "
                    f"{parts[0].dtype}, member {i} has {tuple(p.shape)} {p.dtype}")
        acc = empty_like_layout(parts[0], parts[0].shape)
        _copy_into(acc, parts[0])
        for p in parts[1:]:
            _fold_into(acc, p, op)
        return acc

    def barrier(self, members, me: int) -> None:
        self.gather_meta(members, me, None)


class DistTransport:
    """torch.distributed process groups: NCCL for device payloads, plus a
    gloo twin of every group for small host metadata."""

    def __init__(self, mesh: DeviceMesh, rank: int, backend: str):
        import torch.distributed as dist

        self.dist = dist
        self.kind = backend
        self.rank = rank
        self.mesh = mesh
        # every rank must create every group, in the same order
        self.groups = {}
        self.meta_groups = {}
        self.world_meta = dist.new_group(list(range(mesh.world_size)), backend="gloo")
        for axis in range(mesh.ndim):
            other = [range(mesh.shape[a]) for a in range(mesh.ndim) if a != axis]
            lines = []
            if not other:
                lines.append(tuple(range(mesh.shape[0])))
            else:
                for o in other[0]:
                    coords = [0] * mesh.ndim
                    coords[1 - axis] = o
                    lines.append(mesh.line(coords, axis))
            for line in lines:
                g = dist.new_group(list(line), backend=backend)
                m = g if backend == "gloo" else dist.new_group(list(line), backend="gloo")
                self.groups[line] = g
                self.meta_groups[line] = m

    def exchange_start(self, sends, recvs):
        """Post every send/recv of one exchange round (one NCCL group) and
        return a handle; `wait()` orders the caller's stream after them, so
        device work launched in between overlaps the transfer."""
        dist = self.dist
        ops = []
        keep = []
        after = []
        # gloo carries host tensors: device payloads (the "gloo-cuda" test mesh:
        # several processes on one GPU, where NCCL refuses duplicate devices)
        # are staged through host memory
        stage = self.kind != "nccl"
        for dst, t in sends:
            t = t if _dense(t) else t.contiguous()
            if stage and t.is_cuda:
                t = t.cpu()
            keep.append(t)
            # the wire format is the payload's bytes in memory order: a dense
            # channels-last face travels as-is (a flat view, no transpose)
            ops.append(dist.P2POp(dist.isend, _flat(t), dst))
        for src, out in recvs:
            if stage and out.is_cuda:
                host = torch.empty_strided(out.shape, out.stride(), dtype=out.dtype) \
                    if _dense(out) else torch.empty(out.shape, dtype=out.dtype)
                after.append((out, host))
                out = host
            if not _dense(out):
                raise CollectiveError("receive buffers must be dense")
            ops.append(dist.P2POp(dist.irecv, _flat(out), src))
        if not ops:
            return _Done()
        if self.kind == "nccl":
            return _Pending(dist.batch_isend_irecv(ops), keep)
        return _Pending([op.op(op.tensor, op.peer) for op in ops], keep, after)

    def exchange(self, sends, recvs) -> None:
        self.exchange_start(sends, recvs).wait()

    def gather_meta(self, members, me: int, obj) -> list:
        out = [None] * len(members)
        self.dist.all_gather_object(out, obj, group=self.meta_groups[tuple(members)])
        return out

    def send_meta(self, dst, obj) -> None:
        self.dist.send_object_list([obj], dst=dst, group=self.world_meta)

    def recv_meta(self, src):
        box = [None]
        self.dist.recv_object_list(box, src=src, group=self.world_meta)
        return box[0]

    def all_reduce(self, members, me: int, t: torch.Tensor, op: str) -> torch.Tensor:
        dist = self.dist
        staged = self.kind != "nccl" and t.is_cuda
        out = t.cpu() if staged else t.clone()
        rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
        dist.all_reduce(out, op=rop, group=self.groups[tuple(members)])
        return out.to(t.device) if staged else out

    def barrier(self, members, me: int) -> None:
        self.dist.barrier(group=self.meta_groups[tuple(members)])


class _NcclPending:
    """Handle of one exchange round on the transport's comm stream: wait()
    orders the caller's current stream after it (no host block)."""

    def __init__(self, done, keep):
        self.done = done
        self.keep = keep

    def wait(self) -> None:
        if self.done is not None:
            torch.cuda.current_stream().wait_event(self.done)
        self.done = None
        self.keep = []


class NativeTransport(DistTransport):
    """One process per GPU: the data plane is NCCL through libdpb200.so's C
    ABI (comm.py / csrc/comm.cu) on a dedicated comm stream, the control
    plane (rendezvous, unique-id broadcast, metadata, barriers) is gloo.

    Communicators are created eagerly here — the world communicator for
    every point-to-point round (halo faces, reverse halos, K||V hops,
    redistribute blocks) and one ncclCommSplit per mesh axis for the
    all-reduces — so no exchange round ever depends on a lazily created,
    collective-on-first-use communicator: ranks with nothing to send in a
    round simply post nothing.  Exchange rounds run on the comm stream after
    an event from the caller's stream, and their handle's wait() makes the
    caller's stream wait on the round's completion event, so compute
    launched between post and wait overlaps the transfer.  `timing`, when a
    list, collects (start, end, bytes) CUDA events per round (bench.py)."""

    def __init__(self, mesh: DeviceMesh, rank: int, device, timeout: float):
        super().__init__(mesh, rank, "gloo")
        from . import comm

        self.kind = "nccl"
        self.timeout = timeout
        self.device = torch.device(device)
        box = [comm.unique_id() if rank == 0 else None]
        self.dist.broadcast_object_list(box, src=0, group=self.world_meta)
        self.world = comm.NcclComm.init(mesh.world_size, rank, box[0])
        self.stream = torch.cuda.Stream(device=self.device)
        self.timing = None
        coords = mesh.coords_of(rank)
        self.line_comms = {}
        for axis in range(mesh.ndim):
            line = mesh.line(coords, axis)
            if mesh.ndim == 1:
                self.line_comms[line] = self.world
            else:
                self.line_comms[line] = self.world.split(color=coords[1 - axis],
                                                         key=coords[axis])

    def exchange_start(self, sends, recvs):
        ops, keep = [], []
        for dst, t in sends:
            t = t if _dense(t) else t.contiguous()
            keep.append(t)
            ops.append((dst, False, _flat(t)))
        for src, out in recvs:
            if not _dense(out):
                raise CollectiveError("receive buffers must be dense")
            keep.append(out)
            ops.append((src, True, _flat(out)))
        if not ops:
            return _Done()
        cur = torch.cuda.current_stream(self.device)
        ready = torch.cuda.Event()
        ready.record(cur)
        self.stream.wait_event(ready)
        t0 = t1 = None
        if self.timing is not None:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(self.stream)
        self.world.exchange(ops, self.stream)
        done = torch.cuda.Event(enable_timing=False)
        if t1 is not None:
            t1.record(self.stream)
            self.timing.append((t0, t1, sum(t.numel() * t.element_size() for _, r, t in ops
                                              if not r)))
        done.record(self.stream)
        for t in keep:
            if t.is_cuda:
                t.record_stream(self.stream)
        return _NcclPending(done, keep)

    def exchange(self, sends, recvs) -> None:
        self.exchange_start(sends, recvs).wait()

    def all_reduce(self, members, me: int, t: torch.Tensor, op: str) -> torch.Tensor:
        comm = self.line_comms[tuple(members)]
        src = t if t.is_contiguous() else t.contiguous()
        out = torch.empty_like(src)
        comm.allreduce(src, out, op, torch.cuda.current_stream(self.device))
        return out

    def barrier(self, members, me: int) -> None:
        # watchdog first: every posted round must drain (or raise
        # CollectiveError on an NCCL error / the mesh timeout), then the host
        # rendezvous of the reference's barrier
        self.world.wait(self.stream, self.timeout)
        self.world.wait(torch.cuda.current_stream(self.device), self.timeout)
        super().barrier(members, me)

    def close(self) -> None:
        seen = set()
        for c in list(self.line_comms.values()) + [self.world]:
            if id(c) not in seen and c is not None:
                seen.add(id(c))
                c.destroy()


def _dense(t: torch.Tensor) -> bool:
    """Non-overlapping and dense (some permutation of a contiguous layout)."""
    return t.is_contiguous() or t.is_contiguous(memory_format=memory_format_of(t))


def _fold_into(acc: torch.Tensor, part: torch.Tensor, op: str) -> None:
    """acc = acc (+|max) part: the library's accumulate / max kernels on
    device, host arithmetic for CPU tensors (the gloo test meshes)."""
    if acc.is_cuda:
        from . import kernels

        if op == "sum":
            kernels.accumulate(acc, part)
        else:
            kernels.max_into(acc, part)
    elif op == "sum":
        acc.add_(part)
    else:
        torch.maximum(acc, part, out=acc)


def _flat(t: torch.Tensor) -> torch.Tensor:
    """1-D contiguous view of a dense tensor's memory (element order = memory
    order); the process-group P2P calls require standard contiguity."""
    if t.is_contiguous():
        return t.reshape(-1)
    return t.as_strided((t.numel(),), (1,))


def _copy_into(dst: torch.Tensor, src: torch.Tensor) -> None:
    """Device tensors move through the extension's strided-copy kernel; host
    tensors (CPU/gloo mesh tests) use a host copy."""
    if dst.is_cuda:
        from . import kernels

        kernels.copy_strided(dst, src)
    else:
        dst.copy_(src)


# ---------------------------------------------------------------------------
# rank context and axis groups


class RankContext:
    """Per-rank handle: identity, mesh, device, transport, and the two
    bookkeeping fields the dispatch layer reads (collective_count and a
    bounded trace ring buffer, domainpar/mesh.py:132-151)."""

    def __init__(self, mesh: DeviceMesh, rank_id: int, transport, *, seed: int = 0,
                 device=None):
        self.mesh = mesh
        self.rank_id = int(rank_id)
        self.coords = mesh.coords_of(self.rank_id)
        self.transport = transport
        self.seed = seed
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.collective_count = 0
        self.trace = deque(maxlen=1024)
        self._groups = {}

    def axis_group(self, axis_name: str | None = None) -> "AxisGroup":
        if axis_name is None:
            if self.mesh.ndim != 1:
                raise DimensionError("axis_name is required on a 2-D mesh")
            axis_name = self.mesh.axis_names[0]
        grp = self._groups.get(axis_name)
        if grp is None:
            grp = AxisGroup(self, axis_name)
            self._groups[axis_name] = grp
        return grp

    def __repr__(self):
        return f"RankContext(rank={self.rank_id}, coords={self.coords}, device={self.device})"


class AxisGroup:
    """The ranks along one mesh axis through this rank, in coordinate order."""

    def __init__(self, ctx: RankContext, axis_name: str):
        self.ctx = ctx
        self.axis_name = axis_name
        self.axis = ctx.mesh.axis_index(axis_name)
        self.members = ctx.mesh.line(ctx.coords, self.axis)
        self.index = self.members.index(ctx.rank_id)

    @property
    def size(self) -> int:
        return len(self.members)

    def __repr__(self):
        return f"AxisGroup(axis={self.axis_name!r}, members={self.members})"


# ---------------------------------------------------------------------------
# collectives (public API, reference semantics)


def _count(group: AxisGroup) -> None:
    group.ctx.collective_count += 1


def all_reduce(group: AxisGroup, local: torch.Tensor, op: str = "sum") -> torch.Tensor:
    """Sum or max over the group (domainpar/mesh.py:252-277).  Returns a new
    tensor; the input is not modified."""
    if op not in REDUCE_OPS:
        raise DimensionError(f"all_reduce op must be one of {REDUCE_OPS}, got {op!r}")
    _count(group)
    if group.size == 1:
        return local.clone()
    return group.ctx.transport.all_reduce(group.members, group.index, local, op)


def _narrow(t: torch.Tensor, dim: int, start: int, length: int) -> torch.Tensor:
    return t.narrow(dim, start, length)


def memory_format_of(t: torch.Tensor):
    """The dense memory format `t` is laid out in: channels-last (NHWC /
    NDHWC, the conv hot path's layout) when it is channels-last and not
    plain contiguous, else torch.contiguous_format.  When a tensor satisfies
    both, the two byte layouts coincide."""
    if t.dim() == 5 and not t.is_contiguous() and \
            t.is_contiguous(memory_format=torch.channels_last_3d):
        return torch.channels_last_3d
    if t.dim() == 4 and not t.is_contiguous() and \
            t.is_contiguous(memory_format=torch.channels_last):
        return torch.channels_last
    return torch.contiguous_format


def empty_in_format(shape, fmt, dtype, device) -> torch.Tensor:
    """Uninitialised tensor of `shape` laid out densely in memory format `fmt`."""
    if fmt is torch.contiguous_format or len(shape) != (5 if fmt is torch.channels_last_3d else 4):
        return torch.empty(tuple(shape), dtype=dtype, device=device)
    return torch.empty(tuple(shape), dtype=dtype, device=device, memory_format=fmt)


def empty_like_layout(ref: torch.Tensor, shape, dtype=None) -> torch.Tensor:
    """Allocate `shape` in `ref`'s memory format (channels-last stays
    channels-last, so halo buffers and gradients stay in the layout the
    tcgen05 conv consumes: C innermost, one contiguous run per face)."""
    return empty_in_format(shape, memory_format_of(ref), dtype or ref.dtype, ref.device)


def _packed(t: torch.Tensor, fmt=torch.contiguous_format) -> torch.Tensor:
    """`t` itself when it is one dense run in memory format `fmt`, else a copy
    packed into that format — the halo / varlen pack kernel on device, a host
    copy for CPU tensors.  Sender and receiver agree on `fmt` (the format of
    their local blocks), so a channels-last D/H face (one contiguous run) goes
    out in place with no pack at all."""
    if t.is_contiguous(memory_format=fmt):
        return t
    out = empty_in_format(t.shape, fmt, t.dtype, t.device)
    _copy_into(out, t)
    return out


def gather_known(group: AxisGroup, local: torch.Tensor, dim: int, extents) -> torch.Tensor:
    """Varlen all-gather along `dim` when every member's extent is already
    known (replicated shard_shapes): receives land directly in their slice of
    the output when that slice is contiguous, otherwise in a staging buffer
    that the unpack kernel scatters.  Not counted — callers count."""
    extents = [int(e) for e in extents]
    shape = list(local.shape)
    shape[dim] = sum(extents)
    fmt = memory_format_of(local)
    out = empty_in_format(shape, fmt, local.dtype, local.device)
    me = group.index
    offs = [0]
    for e in extents:
        offs.append(offs[-1] + e)
    mine = _narrow(out, dim, offs[me], extents[me])
    if extents[me]:
        _copy_into(mine, local)
    if group.size == 1:
        return out
    sends = []
    payload = _packed(local, fmt)
    if payload.numel():
        for i, r in enumerate(group.members):
            if i != me:
                sends.append((r, payload))
    recvs = []
    unpack = []
    for i, r in enumerate(group.members):
        if i == me or extents[i] == 0 or out.numel() == 0:
            continue
        dst = _narrow(out, dim, offs[i], extents[i])
        if dst.is_contiguous(memory_format=fmt):
            recvs.append((r, dst))
        else:
            stage = empty_in_format(dst.shape, fmt, out.dtype, out.device)
            recvs.append((r, stage))
            unpack.append((dst, stage))
    group.ctx.transport.exchange(sends, recvs)
    for dst, stage in unpack:
        _copy_into(dst, stage)
    return out


def all_gather_varlen(group: AxisGroup, local: torch.Tensor, dim: int) -> torch.Tensor:
    """Concatenate every member's block along `dim` in member order; extents
    along `dim` may differ (zero included), all other extents and the dtype
    must match (domainpar/mesh.py:280-302)."""
    if not 0 <= dim < local.dim():
        raise DimensionError(f"gather dim {dim} out of range for shape {tuple(local.shape)}")
    _count(group)
    shape = tuple(local.shape)
    info = group.ctx.transport.gather_meta(group.members, group.index,
                                           (shape, str(local.dtype))) \
        if group.size > 1 else [(shape, str(local.dtype))]
    shape0, dt0 = info[0]
    rest0 = tuple(s for a, s in enumerate(shape0) if a != dim)
    for i, (sh, dt) in enumerate(info):
        rest = tuple(s for a, s in enumerate(sh) if a != dim)
        if len(sh) != len(shape0) or rest != rest0 or dt != dt0:
            raise CollectiveError(
                f"all_gather_varlen mismatch off dim {dim}: member 0 has {shape0} {dt0}, "
                f"member {i} has {sh} {dt}")
    return gather_known(group, local, dim, [sh[dim] for sh, _ in info])


def ring_shift_known(group: AxisGroup, payload: torch.Tensor, recv_shape) -> torch.Tensor:
    """Send to index+1, receive a `recv_shape` block from index-1.  Uncounted."""
    r = group.size
    if r == 1:
        return payload
    nxt = group.members[(group.index + 1) % r]
    prv = group.members[(group.index - 1) % r]
    out = torch.empty(tuple(recv_shape), dtype=payload.dtype, device=payload.device)
    sends = [(nxt, _packed(payload))] if payload.numel() else []
    recvs = [(prv, out)] if out.numel() else []
    if group.ctx.transport.kind == "thread":
        # thread mailboxes are FIFO per pair: empty payloads still travel so the
        # pairing of sends and receives never depends on the data
        sends = [(nxt, _packed(payload))]
        recvs = [(prv, out)]
    group.ctx.transport.exchange(sends, recvs)
    return out


def ring_shift(group: AxisGroup, payload: torch.Tensor) -> torch.Tensor:
    """Send to the next member, receive from the previous, wrapping
    (domainpar/mesh.py:305-315).  R=1 is a counted no-op."""
    _count(group)
    if group.size == 1:
        return payload
    shapes = group.ctx.transport.gather_meta(group.members, group.index, tuple(payload.shape))
    return ring_shift_known(group, payload, shapes[(group.index - 1) % group.size])


def halo_sendrecv(group: AxisGroup, local: torch.Tensor, dim: int, serve_left: int,
                  serve_right: int, lw: int, rw: int, *, wait: bool = True):
    """The data phase of a halo exchange with every width already known:
    send my first `serve_left` rows to the previous member and my last
    `serve_right` rows to the next, receive `lw` rows from the previous and
    `rw` rows from the next.  Returns (left_halo, right_halo) as contiguous
    blocks (None when zero-width).  Uncounted.  With wait=False the transfer
    is only posted and a third value, the handle to wait on, is returned."""
    i = group.index
    left = group.members[i - 1] if i > 0 else None
    right = group.members[i + 1] if i < group.size - 1 else None
    extent = local.shape[dim]
    # faces travel and land in the local block's own memory format: a
    # channels-last D (3-D) / H (2-D) face of a batch-1 block is one contiguous
    # run, sent in place, and the received halo is directly a tcgen05 operand
    fmt = memory_format_of(local)
    sends, recvs = [], []
    if left is not None and serve_left > 0:
        sends.append((left, _packed(_narrow(local, dim, 0, serve_left), fmt)))
    if right is not None and serve_right > 0:
        sends.append((right, _packed(_narrow(local, dim, extent - serve_right, serve_right), fmt)))
    lh = rh = None
    if left is not None and lw > 0:
        shp = list(local.shape)
        shp[dim] = lw
        lh = empty_in_format(shp, fmt, local.dtype, local.device)
        recvs.append((left, lh))
    if right is not None and rw > 0:
        shp = list(local.shape)
        shp[dim] = rw
        rh = empty_in_format(shp, fmt, local.dtype, local.device)
        recvs.append((right, rh))
    if not wait:
        return lh, rh, group.ctx.transport.exchange_start(sends, recvs)
    group.ctx.transport.exchange(sends, recvs)
    return lh, rh


def halo_error_text(requester: int, width: int, server: int, extent: int, dim: int) -> str:
    """The reference's HaloError message (domainpar/mesh.py:357-368)."""
    return (f"rank {requester} requested halo width {width} from rank {server}, "
            f"which holds only {extent} along dim {dim} (halos are single-hop)")


def halo_exchange(group: AxisGroup, local: torch.Tensor, dim: int, left_width: int,
                  right_width: int) -> torch.Tensor:
    """Extend `local` with `left_width` rows from the previous member and
    `right_width` rows from the next along `dim` (non-periodic; the ends get
    nothing).  A request wider than the holder's extent is a HaloError raised
    on the serving rank (domainpar/mesh.py:318-386).  One metadata round
    replaces the reference's width handshake; it is part of this one
    collective."""
    if not 0 <= dim < local.dim():
        raise DimensionError(f"halo dim {dim} out of range for shape {tuple(local.shape)}")
    if left_width < 0 or right_width < 0:
        raise DimensionError(f"halo widths must be >= 0, got ({left_width}, {right_width})")
    _count(group)
    ctx = group.ctx
    i, n = group.index, group.size
    extent = int(local.shape[dim])
    lw = left_width if i > 0 else 0
    rw = right_width if i < n - 1 else 0
    if n == 1:
        return local
    info = ctx.transport.gather_meta(group.members, i, (int(left_width), int(right_width), extent))
    # every rank sees every request; the server raises the reference's text,
    # everybody else unwinds without touching the device
    problems = []
    for m in range(n):
        ml, mr, _ = info[m]
        if m + 1 < n and mr > info[m + 1][2]:
            problems.append((group.members[m], mr, m + 1))
        if m > 0 and ml > info[m - 1][2]:
            problems.append((group.members[m], ml, m - 1))
    for requester, width, server in problems:
        if server == i:
            raise HaloError(halo_error_text(requester, width, ctx.rank_id, extent, dim))
    if problems:
        raise PeerAbort(f"rank {ctx.rank_id}: unwinding, another rank failed")
    serve_left = info[i - 1][1] if i > 0 else 0
    serve_right = info[i + 1][0] if i < n - 1 else 0
    lh, rh = halo_sendrecv(group, local, dim, serve_left, serve_right, lw, rw)
    if lh is None and rh is None:
        return local
    shp = list(local.shape)
    shp[dim] = lw + extent + rw
    out = empty_like_layout(local, shp)
    pos = 0
    for piece in (lh, local, rh):
        if piece is None:
            continue
        w = piece.shape[dim]
        if w:
            _copy_into(_narrow(out, dim, pos, w), piece)
        pos += w
    return out


def barrier(group: AxisGroup) -> None:
    """Block until every member arrives (domainpar/mesh.py:389-403)."""
    _count(group)
    if group.size > 1:
        group.ctx.transport.barrier(group.members, group.index)


# ---------------------------------------------------------------------------
# launchers


def _default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")


def _raise_mesh_error(failures: dict):
    primaries = {r: e for r, e in failures.items() if not isinstance(e, PeerAbort)}
    if not primaries:
        primaries = failures
    detail = "; ".join(f"rank {r}: {type(e).__name__}: {e}" for r, e in sorted(primaries.items()))
    err = MeshError(f"{len(primaries)} rank(s) failed: {detail}", failures=failures)
    raise err from next(iter(primaries.values()))


def _spawn_threads(mesh: DeviceMesh, fn, seed: int, timeout: float, device):
    rt = _ThreadRuntime(mesh, timeout)
    n = mesh.world_size
    results = [None] * n
    failures = {}
    lock = threading.Lock()
    dev = torch.device(device) if device is not None else _default_device()
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())

    def run(rank: int):
        try:
            if dev.type == "cuda":
                torch.cuda.set_device(dev)
            ctx = RankContext(mesh, rank, ThreadTransport(rt, rank), seed=seed, device=dev)
            results[rank] = fn(ctx)
        except BaseException as exc:  # noqa: BLE001 - surfaced through MeshError
            with lock:
                failures[rank] = exc
            rt.abort.set()
        finally:
            rt.finished[rank].set()

    threads = [threading.Thread(target=run, args=(r,), name=f"dp-rank-{r}") for r in range(n)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if failures:
        _raise_mesh_error(failures)
    return results


def _to_host(value):
    if isinstance(value, torch.Tensor):
        return value.detach().cpu()
    if isinstance(value, (list, tuple)):
        return type(value)(_to_host(v) for v in value)
    if isinstance(value, dict):
        return {k: _to_host(v) for k, v in value.items()}
    return value


def _proc_main(rank, world, port, mesh_shape, names, fn, seed, timeout, backend, out_q):
    import datetime
    import pickle

    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        on_gpu = backend in ("nccl", "gloo-cuda")
        native = backend == "nccl" and os.environ.get("DP_TRANSPORT", "native") != "torch"
        pg_backend = "gloo" if (backend == "gloo-cuda" or native) else backend
        if on_gpu:
            torch.cuda.set_device(rank % torch.cuda.device_count())
        dist.init_process_group(pg_backend, rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=max(timeout, 1.0)))
        mesh = DeviceMesh(mesh_shape, names)
        dev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
        tr = NativeTransport(mesh, rank, dev, timeout) if native else \
            DistTransport(mesh, rank, pg_backend)
        ctx = RankContext(mesh, rank, tr, seed=seed, device=dev)
        res = _to_host(fn(ctx))
        out_q.put((rank, "ok", pickle.dumps(res)))
    except BaseException as exc:  # noqa: BLE001
        try:
            out_q.put((rank, "err", pickle.dumps(exc)))
        except Exception:  # unpicklable exception
            out_q.put((rank, "err", pickle.dumps(CollectiveError(f"{type(exc).__name__}: {exc}"))))
    finally:
        try:
            close = getattr(getattr(locals().get("ctx"), "transport", None), "close", None)
            if close is not None:
                close()
            if dist.is_initialized():
                dist.destroy_process_group()
        except Exception:
            pass


def _spawn_procs(mesh: DeviceMesh, fn, seed: int, timeout: float, backend: str):
    import pickle
    import socket

    import torch.multiprocessing as mp

    n = mesh.world_size
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_main,
                         args=(r, n, port, mesh.shape, mesh.axis_names, fn, seed, timeout,
                               backend, q))
             for r in range(n)]
    for p in procs:
        p.start()
    results = [None] * n
    failures = {}
    got = 0
    deadline = time.monotonic() + timeout + 120.0
    while got < n:
        try:
            rank, status, blob = q.get(timeout=1.0)
        except queue.Empty:
            if time.monotonic() > deadline or all(not p.is_alive() for p in procs):
                for r in range(n):
                    if results[r] is None and r not in failures:
                        failures[r] = CollectiveError(f"rank {r} exited without a result")
                break
            continue
        got += 1
        if status == "ok":
            results[rank] = pickle.loads(blob)
        else:
            failures[rank] = pickle.loads(blob)
    for p in procs:
        p.join(timeout=10)
        if p.is_alive():
            p.kill()
    if failures:
        _raise_mesh_error(failures)
    return results


def spawn_mesh(shape, axis_names, fn, *, seed: int = 0, timeout: float | None = None,
               backend: str = "thread", device=None):
    """Run fn(ctx) on every rank of a fresh mesh; return results by rank id.

    backend "thread" (default, the reference's model — domainpar/mesh.py:420)
    runs every rank as a thread of this process on `device` (default: the
    current CUDA device, else CPU).  "nccl" launches one process per GPU,
    "gloo" one CPU process per rank, and "gloo-cuda" one process per rank that
    all share the GPU (device payloads staged through host memory: the
    multi-process path with real kernels on a one-GPU box); their fn must be
    picklable and results
    come back on the host.  Any rank failing surfaces as one MeshError naming
    the primary failure(s).
    """
    mesh = DeviceMesh(tuple(shape), tuple(axis_names))
    tmo = _resolve_timeout(timeout)
    if backend == "thread":
        return _spawn_threads(mesh, fn, seed, tmo, device)
    if backend in ("nccl", "gloo", "gloo-cuda"):
        return _spawn_procs(mesh, fn, seed, tmo, backend)
    raise DimensionError(f"unknown mesh backend {backend!r}")


def init_mesh(shape=None, axis_names=("domain",), *, seed: int = 0,
              backend: str | None = None) -> RankContext:
    """Production entry under torchrun: join the already-launched world
    (RANK / WORLD_SIZE / MASTER_* from the environment), one process per GPU,
    and return this process's RankContext."""
    import datetime

    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if backend is None:
        # DP_MESH_BACKEND=gloo-cuda: ranks share the visible GPU(s) over gloo
        # (a multi-process dry run of the N-GPU path on a one-GPU box)
        backend = os.environ.get("DP_MESH_BACKEND") or (
            "nccl" if torch.cuda.is_available() else "gloo")
    if shape is None:
        shape = (world,)
    mesh = DeviceMesh(tuple(shape), tuple(axis_names))
    if mesh.world_size != world:
        raise DimensionError(f"mesh {mesh.shape} needs {mesh.world_size} ranks, world is {world}")
    gpu_gloo = backend == "gloo-cuda"
    if gpu_gloo:
        backend = "gloo"
        local = local % torch.cuda.device_count()
    if backend == "nccl" or gpu_gloo:
        torch.cuda.set_device(local)
    # DP_TRANSPORT=torch keeps torch.distributed's NCCL process groups as the
    # data plane instead of the library's own communicators
    native = backend == "nccl" and os.environ.get("DP_TRANSPORT", "native") != "torch"
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo" if native else backend, rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=_resolve_timeout(None) * 20))
    dev = torch.device("cuda", local) if (backend == "nccl" or gpu_gloo) else torch.device("cpu")
    if native:
        tr = NativeTransport(mesh, rank, dev, _resolve_timeout(None))
    else:
        tr = DistTransport(mesh, rank, backend)
    return RankContext(mesh, rank, tr, seed=seed, device=dev)
