"""Attention restated from the reference (TEST INFRASTRUCTURE).

sdpa()        domainpar/dense.py:223-234,258-271 — fp64 max-shifted softmax
RingState     domainpar/ops.py:180-214 — fp64 online softmax (m, l, acc)
ring_members()  per-member outputs of domainpar/ops.py:217-279: member i
              folds K/V blocks in ring order (i, i-1, i-2, ...)
sdpa_grads()  analytic gradients in fp64 (no reference function; pinned by
              finite differences in tests/test_oracle.py)
head_slab()   one head's output / dq on a query-row slab and dk / dv on a
              key slab at full sequence length, the same formulas restricted
              (row statistics LSE / delta for every query computed in chunks):
              full-size parity; pinned against sdpa / sdpa_grads.
Multi-head inputs [S, H, d] are handled head by head (the reference is
single-head [S, d]; its ViT pipeline loops heads, ops.py:590-600).
"""

import math

import numpy as np


def softmax64(s):
    s = s.astype(np.float64)
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def _heads(t):
    return t[:, None, :] if t.ndim == 2 else t


def sdpa(q, k, v):
    q3, k3, v3 = _heads(q), _heads(k), _heads(v)
    scale = 1.0 / math.sqrt(q.shape[-1])
    out = np.empty(q3.shape, dtype=np.float64)
    for h in range(q3.shape[1]):
        s = (q3[:, h].astype(np.float64) @ k3[:, h].astype(np.float64).T) * scale
        out[:, h] = softmax64(s) @ v3[:, h].astype(np.float64)
    out = out.astype(q.dtype)
    return out if q.ndim == 3 else out[:, 0]


class RingState:
    def __init__(self, rows, d):
        self.m = np.full(rows, -np.inf)
        self.l = np.zeros(rows)
        self.acc = np.zeros((rows, d))

    def update(self, s, v):
        if s.shape[1] == 0:
            return
        s = s.astype(np.float64)
        v = v.astype(np.float64)
        m_new = np.maximum(self.m, s.max(axis=1))
        c = np.exp(self.m - m_new)
        p = np.exp(s - m_new[:, None])
        self.l = self.l * c + p.sum(axis=1)
        self.acc = self.acc * c[:, None] + p @ v
        self.m = m_new

    def output(self):
        return self.acc / self.l[:, None]


def ring_members(q, k, v, q_ext, kv_ext):
    """Per-member outputs (member order) of the ring algorithm."""
    r = len(q_ext)
    qb = np.concatenate([[0], np.cumsum(q_ext)]).astype(int)
    kb = np.concatenate([[0], np.cumsum(kv_ext)]).astype(int)
    q3, k3, v3 = _heads(q), _heads(k), _heads(v)
    scale = 1.0 / math.sqrt(q.shape[-1])
    outs = []
    for i in range(r):
        ql = q3[qb[i]:qb[i + 1]]
        o = np.empty(ql.shape, dtype=np.float64)
        for h in range(q3.shape[1]):
            st = RingState(ql.shape[0], q.shape[-1])
            for t in range(r):
                j = (i - t) % r
                kl = k3[kb[j]:kb[j + 1], h]
                vl = v3[kb[j]:kb[j + 1], h]
                if kl.shape[0]:
                    st.update((ql[:, h].astype(np.float64) @ kl.astype(np.float64).T) * scale, vl)
            o[:, h] = st.output() if ql.shape[0] else np.zeros((0, q.shape[-1]))
        o = o.astype(q.dtype)
        outs.append(o if q.ndim == 3 else o[:, 0])
    return outs


def sdpa_grads(q, k, v, do):
    """(dq, dk, dv) of out = sdpa(q, k, v) given dO, in float64."""
    q3, k3, v3, d3 = (_heads(t).astype(np.float64) for t in (q, k, v, do))
    scale = 1.0 / math.sqrt(q.shape[-1])
    dq, dk, dv = np.zeros_like(q3), np.zeros_like(k3), np.zeros_like(v3)
    for h in range(q3.shape[1]):
        p = softmax64(q3[:, h] @ k3[:, h].T * scale)
        o = p @ v3[:, h]
        dv[:, h] = p.T @ d3[:, h]
        dp = d3[:, h] @ v3[:, h].T
        delta = (d3[:, h] * o).sum(axis=1, keepdims=True)
        ds = p * (dp - delta)
        dq[:, h] = ds @ k3[:, h] * scale
        dk[:, h] = ds.T @ q3[:, h] * scale
    if q.ndim == 2:
        return dq[:, 0], dk[:, 0], dv[:, 0]
    return dq, dk, dv


def head_slab(q, k, v, do, rows, keys, chunk=2048):
    """One head ([S, d] arrays): (o[rows], dq[rows], dk[keys], dv[keys]) of
    sdpa with dO, at any S.  Query rows need all keys (fp64, rows x S);
    the key slab needs every query's LSE and delta = rowsum(dO * O), taken
    chunk by chunk (scores of a chunk in fp32 BLAS, exp / sums in fp64)."""
    S, d = q.shape
    scale = 1.0 / math.sqrt(d)
    q64, k64, v64, d64 = (t.astype(np.float64) for t in (q, k, v, do))
    # query-row slab
    p = softmax64(q64[rows] @ k64.T * scale)
    o = p @ v64
    dp = d64[rows] @ v64.T
    delta = (d64[rows] * o).sum(axis=1, keepdims=True)
    dq = (p * (dp - delta)) @ k64 * scale
    # every query's lse and delta
    q32, k32, v32 = (t.astype(np.float32) for t in (q, k, v))
    lse = np.empty(S)
    dl = np.empty(S)
    for c0 in range(0, S, chunk):
        s = (q32[c0:c0 + chunk] @ k32.T).astype(np.float64) * scale
        mx = s.max(axis=1, keepdims=True)
        e = np.exp(s - mx)
        den = e.sum(axis=1, keepdims=True)
        lse[c0:c0 + chunk] = (mx + np.log(den))[:, 0]
        oc = (e / den).astype(np.float32) @ v32
        dl[c0:c0 + chunk] = (d64[c0:c0 + chunk] * oc.astype(np.float64)).sum(axis=1)
    # key slab
    pk = np.exp(q64 @ k64[keys].T * scale - lse[:, None])        # [S, |keys|]
    dpk = d64 @ v64[keys].T
    dsk = pk * (dpk - dl[:, None])
    dv = pk.T @ d64
    dk = dsk.T @ q64 * scale
    return o, dq, dk, dv
