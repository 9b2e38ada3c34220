"""Integer planning restated from the reference (TEST INFRASTRUCTURE).

default_chunk         domainpar/sharding.py:83-103
owned_output_range    domainpar/ops.py:286-300
halo widths           domainpar/ops.py:363-385
trim / pad            domainpar/ops.py:397-413
"""

import math


def default_chunk(extent, members):
    # sharding.py:94-103 — ceil-sized pieces, remainder, zeros
    if extent == 0:
        return [0] * members
    c = math.ceil(extent / members)
    out, rem = [], extent
    for _ in range(members):
        t = min(c, rem)
        out.append(t)
        rem -= t
    return out


def conv_out(g, k, s, p):
    # dense.py:142-150
    n = (g + 2 * p - k) // s + 1
    if n < 1:
        raise ValueError(f"conv output extent {n} < 1")
    return n


def owned_range(a, b, g_in, g_out, k, s, p):
    # ops.py:293-300
    def first(t):
        if t <= 0:
            return 0
        if t >= g_in:
            return g_out
        return min(g_out, max(0, math.ceil((t + p) / s)))
    return first(a), first(b)


def member_plans(extents, g_in, k, s, p):
    """[(j_lo, j_hi, w_min, w_max, lw, rw)] per member (ops.py:363-385)."""
    g_out = conv_out(g_in, k, s, p)
    bounds = [0]
    for e in extents:
        bounds.append(bounds[-1] + e)
    out = []
    for m in range(len(extents)):
        a, b = bounds[m], bounds[m + 1]
        j_lo, j_hi = owned_range(a, b, g_in, g_out, k, s, p)
        if j_hi > j_lo:
            w_min = j_lo * s - p
            w_max = (j_hi - 1) * s - p + k
            lw = max(0, a - max(w_min, 0))
            rw = max(0, min(w_max, g_in) - b)
        else:
            w_min = w_max = None
            lw = rw = 0
        out.append((j_lo, j_hi, w_min, w_max, lw, rw))
    return out
