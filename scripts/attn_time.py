"""Time one tcgen05 attention fwd block and one bwd block (S x S x 16 heads,
d = 64) with CUDA events; DP_ATTN_DBG selects profiling ablations."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

S = int(os.environ.get("S", "16384"))
H, d = 16, 64
dev = torch.device("cuda", 0)
torch.manual_seed(0)
q, k, v, do = (torch.randn(S, H, d, device=dev).to(torch.bfloat16) for _ in range(4))
m = torch.full((S, H), -math.inf, device=dev)
l = torch.zeros((S, H), device=dev)
acc = torch.zeros((S, H, d), device=dev)
kernels.set_algo("tc")
lse = torch.randn(S, H, device=dev) + 10
delta = torch.randn(S, H, device=dev)
dq = torch.zeros((S, H, d), device=dev)
dk = torch.zeros_like(dq)
dv = torch.zeros_like(dq)


def t(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


f = 4.0 * S * S * d * H
tf = t(lambda: kernels.attn_fwd_update(q, k, v, m, l, acc, 0.125))
tb = t(lambda: kernels.attn_bwd_update(q, k, v, do, lse, delta, dq, dk, dv, 0.125))
print(f"S={S} dbg={os.environ.get('DP_ATTN_DBG', '0')}: fwd {tf:.3f} ms {f / tf / 1e9:.0f} TF/s; "
      f"bwd {tb:.3f} ms {2.5 * f / tb / 1e9:.0f} TF/s")
