"""Small forced-tcgen05 attention forward cases vs fp64 (debug helper)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

dev = torch.device("cuda", 0)
kernels.set_algo("tc")
for sq, sk, H in [(128, 64, 1), (128, 128, 1), (128, 192, 1), (256, 256, 1), (300, 333, 2),
                  (1000, 1000, 2)]:
    torch.manual_seed(0)
    q, k, v = (torch.randn(n, H, 64, device=dev).to(torch.bfloat16) for n in (sq, sk, sk))
    m = torch.full((sq, H), -math.inf, device=dev)
    l = torch.zeros((sq, H), device=dev)
    acc = torch.zeros((sq, H, 64), device=dev)
    kernels.attn_fwd_update(q, k, v, m, l, acc, 0.125)
    out = torch.empty_like(q)
    lse = torch.empty_like(m)
    kernels.attn_finalize(q, m, l, acc, out, lse, 1.0)
    torch.cuda.synchronize()
    ref = torch.softmax(torch.einsum("qhd,khd->hqk", q.double(), k.double()) * 0.125, -1)
    ref = torch.einsum("hqk,khd->qhd", ref, v.double())
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    print(sq, sk, H, "rel err", err, "nan acc", torch.isnan(acc).any().item(),
          "nan l", torch.isnan(l).any().item(), flush=True)
