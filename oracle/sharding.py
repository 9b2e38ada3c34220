"""Layouts of scatter / full_tensor / redistribute restated from the
reference (TEST INFRASTRUCTURE): domainpar/sharding.py:273-384."""

import numpy as np

from .plan import default_chunk


def blocks(g, dim, extents):
    """Member blocks of g split along `dim` (sharding.py:325-332)."""
    b = np.concatenate([[0], np.cumsum(extents)]).astype(int)
    idx = [slice(None)] * g.ndim
    out = []
    for m in range(len(extents)):
        idx[dim] = slice(b[m], b[m + 1])
        out.append(np.ascontiguousarray(g[tuple(idx)]))
    return out


def reshard_1d(g, old_dim, new_dim, members):
    """Shard(old)->Shard(new) on a 1-D mesh = gather then default_chunk
    slice of the new dim (sharding.py:370-383): returns the member blocks
    and the new extents."""
    ext = default_chunk(g.shape[new_dim], members)
    return blocks(g, new_dim, ext), tuple(ext)
