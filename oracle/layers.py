"""Normalisations, linear and the ViT pipeline restated from the reference
(TEST INFRASTRUCTURE — only tests/, smoke() and bench.py's CPU leg use it).

softmax()      domainpar/dense.py:223-234 / ops.py:126-150 — the sharded
               version all-reduces exactly these max / denominator terms,
               so one dense fp64 formula covers both
layer_norm()   domainpar/dense.py:237-255 / ops.py:153-173 — fp64 moments
               E[x^2] - mean^2, clamped at 0
linear()       domainpar/dense.py:101-116
vit_dense()    domainpar/ops.py:615-655 (vit_block_pipeline_dense): patch
               conv -> tokens -> n_layers x (LN, q/k/v, per-head sdpa, proj,
               residual, LN, 2-layer MLP, residual)
vit_weights()  domainpar/ops.py:485-510 — the same NumPy draws
Pinned against the reference's own outputs (tests/golden/layer_cases.npz,
made by tests/golden/make_golden.py) in tests/test_oracle.py.
"""

import numpy as np

from .attention import sdpa
from .conv import conv


def softmax(x, dim):
    x64 = x.astype(np.float64)
    e = np.exp(x64 - x64.max(axis=dim, keepdims=True))
    return (e / e.sum(axis=dim, keepdims=True)).astype(x.dtype)


def layer_norm(x, dim, eps=1e-5):
    x64 = x.astype(np.float64)
    mean = x64.mean(axis=dim, keepdims=True)
    var = np.maximum((x64 * x64).mean(axis=dim, keepdims=True) - mean * mean, 0.0)
    return ((x64 - mean) / np.sqrt(var + eps)).astype(x.dtype)


def linear(x, w, b):
    return x @ w.T + b


def vit_weights(embed_dim, image_channels, patch, n_layers, mlp_hidden, seed=0,
                dtype=np.float32):
    rng = np.random.default_rng(seed)
    d, h = embed_dim, mlp_hidden

    def w(*shape):
        return (rng.standard_normal(shape) * 0.05).astype(dtype)

    out = {"tokenizer": w(d, image_channels, patch, patch)}
    for i in range(n_layers):
        for name, shape in (("wq", (d, d)), ("bq", (d,)), ("wk", (d, d)), ("bk", (d,)),
                            ("wv", (d, d)), ("bv", (d,)), ("wo", (d, d)), ("bo", (d,)),
                            ("w1", (h, d)), ("b1", (h,)), ("w2", (d, h)), ("b2", (d,))):
            out[f"layers.{i}.{name}"] = w(*shape)
    return out


def vit_dense(x, weights, patch, n_layers, n_heads, eps=1e-5):
    tokens = conv(x, weights["tokenizer"], patch, 0)
    c = tokens.shape[0]
    seq = np.ascontiguousarray(np.transpose(tokens, (1, 2, 0)).reshape(-1, c))
    dh = c // n_heads
    for i in range(n_layers):
        p = f"layers.{i}."
        normed = layer_norm(seq, 1, eps)
        q = linear(normed, weights[p + "wq"], weights[p + "bq"])
        k = linear(normed, weights[p + "wk"], weights[p + "bk"])
        v = linear(normed, weights[p + "wv"], weights[p + "bv"])
        attn = np.concatenate([sdpa(q[:, h * dh:(h + 1) * dh], k[:, h * dh:(h + 1) * dh],
                                    v[:, h * dh:(h + 1) * dh]) for h in range(n_heads)], axis=1)
        seq = seq + linear(attn, weights[p + "wo"], weights[p + "bo"])
        normed2 = layer_norm(seq, 1, eps)
        hidden = linear(normed2, weights[p + "w1"], weights[p + "b1"])
        seq = seq + linear(hidden, weights[p + "w2"], weights[p + "b2"])
    return seq
