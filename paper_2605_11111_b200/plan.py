"""Integer planning for the domain-parallel path (host side, no device sync).

Everything here is pure Python integer arithmetic on *replicated*
metadata: every rank can evaluate every member's plan, which is what lets the
device path size each NCCL message locally instead of running the
reference's width handshake (domainpar/mesh.py:347-355).  Parity with the
reference is bit-exact and is checked against integers captured from the
reference itself (tests/golden/plans.json).

Rows of SURVEY.md §8(a) implemented here:
  A1  default_chunk            domainpar/sharding.py:83-103
  A6  owned_output_range       domainpar/ops.py:286-300
      halo_conv_plan           domainpar/ops.py:343-385 (+ trim/pad :397-413)
  A5  redistribute_plan        domainpar/sharding.py:350-384
  A12 ring_source              domainpar/mesh.py:305-315 (send +1, recv -1)
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import DimensionError, ShapeError

__all__ = [
    "default_chunk",
    "prefix_bounds",
    "conv_output_extent",
    "owned_output_range",
    "MemberHaloPlan",
    "HaloConvPlan",
    "halo_conv_plan",
    "ring_source",
]


def default_chunk(extent: int, members: int) -> list[int]:
    """Ceil-sized chunks, then the remainder, then zeros; always `members`
    entries (domainpar/sharding.py:83-103).  (10,4)->[3,3,3,1],
    (5,4)->[2,2,1,0], (0,3)->[0,0,0].  Neither torch.chunk nor
    torch.tensor_split reproduces this."""
    extent = int(extent)
    members = int(members)
    if extent < 0:
        raise DimensionError(f"extent must be >= 0, got {extent}")
    if members < 1:
        raise DimensionError(f"members must be >= 1, got {members}")
    if extent == 0:
        return [0] * members
    size = -(-extent // members)  # exact integer ceil
    out = []
    left = extent
    for _ in range(members):
        piece = size if left >= size else left
        out.append(piece)
        left -= piece
    return out


def prefix_bounds(extents) -> list[int]:
    """[0, e0, e0+e1, ...] — member m owns [bounds[m], bounds[m+1])."""
    bounds = [0]
    for e in extents:
        bounds.append(bounds[-1] + int(e))
    return bounds


def conv_output_extent(extent: int, kernel: int, stride: int, padding: int) -> int:
    """floor((G + 2p - k)/s) + 1, ShapeError when < 1 (domainpar/dense.py:142-150)."""
    n = (extent + 2 * padding - kernel) // stride + 1
    if n < 1:
        raise ShapeError(
            f"conv output extent {n} < 1 for input {extent}, kernel {kernel}, "
            f"stride {stride}, padding {padding}"
        )
    return n


def owned_output_range(a: int, b: int, g_in: int, g_out: int, kernel: int,
                       stride: int, padding: int) -> tuple[int, int]:
    """Output indices j whose anchor clamp(j*s - p, 0, g_in-1) lies in [a, b).

    Restates domainpar/ops.py:286-300.  The anchors are monotone in j, so
    the owned set is the half-open range [first(a), first(b)) where first(t)
    is the smallest j with anchor >= t.
    """
    def first(t: int) -> int:
        if t <= 0:
            return 0
        if t >= g_in:
            return g_out
        # smallest j with j*s - p >= t  ->  ceil((t + p) / s)
        j = -(-(t + padding) // stride)
        return min(g_out, max(0, j))

    return first(a), first(b)


@dataclass(frozen=True)
class MemberHaloPlan:
    """One member's share of a halo convolution along the sharded dim.

    All indices are global along the sharded dim.  The member computes
    output rows [j_lo, j_hi); their windows read input rows
    [w_min, w_max) (w_min may be < 0, w_max may be > G: virtual zeros).
    It owns input rows [a, b) and needs `lw` rows from the previous member
    (always 0 under this ownership rule) and `rw` rows from the next one.

    `base` = w_min - a is where output row 0's window starts relative to
    the first local row: the device kernels index the sharded dim of the
    virtual block  [zeros | local (b-a rows) | right halo (rw rows) | zeros]
    as `base + jj*stride + tap`, which is exactly the reference's trimmed
    and zero-padded block (domainpar/ops.py:397-413) without materialising
    it.
    """

    member: int
    a: int
    b: int
    j_lo: int
    j_hi: int
    w_min: int
    w_max: int
    lw: int
    rw: int

    @property
    def n_out(self) -> int:
        return self.j_hi - self.j_lo

    @property
    def extent(self) -> int:
        return self.b - self.a

    @property
    def base(self) -> int:
        return self.w_min - self.a

    def trim(self, g_in: int) -> tuple[int, int]:
        """[need_lo, need_hi) of the reference's trim (ops.py:400-406)."""
        return max(self.w_min, 0), min(self.w_max, g_in)

    def pads(self, g_in: int) -> tuple[int, int]:
        """Zero rows the reference np.pad's onto the trimmed block (ops.py:407-410)."""
        if self.n_out == 0:
            return 0, 0
        return max(0, -self.w_min), max(0, self.w_max - g_in)


@dataclass(frozen=True)
class HaloConvPlan:
    g_in: int
    g_out: int
    kernel: int
    stride: int
    padding: int
    members: tuple[MemberHaloPlan, ...]

    @property
    def out_extents(self) -> tuple[int, ...]:
        return tuple(m.n_out for m in self.members)

    def served_right(self, member: int) -> int:
        """Rows member `member` must send to member-1 (its left neighbour's rw)."""
        return self.members[member - 1].rw if member > 0 else 0

    def served_left(self, member: int) -> int:
        """Rows member `member` must send to member+1 (that member's lw)."""
        if member + 1 < len(self.members):
            return self.members[member + 1].lw
        return 0

    def hop_violations(self) -> list[tuple[int, int, int, int]]:
        """(requester, width, server, server_extent) for every request a
        single-hop exchange cannot serve (domainpar/mesh.py:357-368)."""
        bad = []
        n = len(self.members)
        for m in self.members:
            if m.rw > 0 and m.member + 1 < n:
                srv = self.members[m.member + 1]
                if m.rw > srv.extent:
                    bad.append((m.member, m.rw, srv.member, srv.extent))
            if m.lw > 0 and m.member > 0:
                srv = self.members[m.member - 1]
                if m.lw > srv.extent:
                    bad.append((m.member, m.lw, srv.member, srv.extent))
        return bad


def halo_conv_plan(in_extents, g_in: int, kernel: int, stride: int,
                   padding: int) -> HaloConvPlan:
    """Per-member ownership + halo widths (domainpar/ops.py:363-385).

    lw is identically 0 under the anchor-ownership rule and rw <= k-1
    (SURVEY.md A6); both are still computed by the reference's formulas so
    the parity test exercises the general case.
    """
    g_out = conv_output_extent(g_in, kernel, stride, padding)
    bounds = prefix_bounds(in_extents)
    if bounds[-1] != g_in:
        raise ShapeError(f"extents {tuple(in_extents)} do not tile {g_in}")
    plans = []
    for m in range(len(in_extents)):
        a, b = bounds[m], bounds[m + 1]
        j_lo, j_hi = owned_output_range(a, b, g_in, g_out, kernel, stride, padding)
        if j_hi > j_lo:
            w_min = j_lo * stride - padding
            w_max = (j_hi - 1) * stride - padding + kernel
            lw = max(0, a - max(w_min, 0))
            rw = max(0, min(w_max, g_in) - b)
        else:
            # an empty member still joins the exchange round; its window is
            # irrelevant, keep it at its own start so `base` is 0
            w_min = w_max = a
            lw = rw = 0
        plans.append(MemberHaloPlan(m, a, b, j_lo, j_hi, w_min, w_max, lw, rw))
    return HaloConvPlan(g_in, g_out, kernel, stride, padding, tuple(plans))


def ring_source(index: int, step: int, size: int) -> int:
    """Member whose K/V block member `index` holds at ring step `step`
    (send to index+1, receive from index-1; domainpar/mesh.py:313-314)."""
    return (index - step) % size
