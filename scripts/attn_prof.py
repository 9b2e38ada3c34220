"""One tcgen05 attention fwd block and one bwd block at a cfg3 ring-step
size (16k x 16k x 16 heads) — a short command for `ncu --set full`."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

S = int(os.environ.get("S", "16384"))
H, d = 16, 64
dev = torch.device("cuda", 0)
q, k, v, do = (torch.randn(S, H, d, device=dev).to(torch.bfloat16) for _ in range(4))
m = torch.full((S, H), -math.inf, device=dev)
l = torch.zeros((S, H), device=dev)
acc = torch.zeros((S, H, d), device=dev)
kernels.set_algo("tc")
kernels.attn_fwd_update(q, k, v, m, l, acc, 0.125)
lse = torch.randn(S, H, device=dev) + 10
delta = torch.randn(S, H, device=dev)
dq = torch.zeros((S, H, d), device=dev)
dk = torch.zeros_like(dq)
dv = torch.zeros_like(dq)
kernels.attn_bwd_update(q, k, v, do, lse, delta, dq, dk, dv, 0.125)
torch.cuda.synchronize()
print("ok")
