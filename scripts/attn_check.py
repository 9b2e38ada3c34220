"""Check + time the tcgen05 attention block kernel against the CUDA-core
kernel and an fp64 reference (GPU helper, not part of the test suite).

    python scripts/attn_check.py [S] [H] [blocks]
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 3
d = 64
dev = torch.device("cuda", 0)
torch.manual_seed(0)
q, k, v = (torch.randn(S, H, d, device=dev).to(torch.bfloat16) for _ in range(3))
scale = 1.0 / math.sqrt(d)


def run(algo, qq, kk, vv):
    kernels.set_algo(algo)
    m = torch.full((qq.shape[0], H), -math.inf, device=dev)
    l = torch.zeros((qq.shape[0], H), device=dev)
    acc = torch.zeros((qq.shape[0], H, d), device=dev)
    cuts = [round(i * kk.shape[0] / nb) for i in range(nb + 1)]
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b > a:
            kernels.attn_fwd_update(qq, kk[a:b], vv[a:b], m, l, acc, scale)
    out = torch.empty_like(qq)
    lse = torch.empty_like(m)
    kernels.attn_finalize(qq, m, l, acc, out, lse, 1.0)
    return out, lse


ref = torch.softmax((q.double().transpose(0, 1) @ k.double().transpose(0, 1).transpose(1, 2)) * scale,
                    -1) @ v.double().transpose(0, 1)
ref = ref.transpose(0, 1)
o_tc, lse_tc = run("tc", q, k, v)
o_si, lse_si = run("simt", q, k, v)
den = ref.abs().max().item()
print(f"S={S} H={H} blocks={nb}: rel err tc {(o_tc.double() - ref).abs().max().item() / den:.3e} "
      f"simt {(o_si.double() - ref).abs().max().item() / den:.3e} "
      f"lse diff {(lse_tc - lse_si).abs().max().item():.3e}")

# timing at a cfg3-like block: 65536 / R queries x keys
for (sq, sk) in ((8192, 8192), (16384, 16384), (65536, 65536)):
    Hh = 16
    qq, kk, vv = (torch.randn(sq if i == 0 else sk, Hh, d, device=dev).to(torch.bfloat16)
                  for i in range(3))
    m = torch.full((sq, Hh), -math.inf, device=dev)
    l = torch.zeros((sq, Hh), device=dev)
    acc = torch.zeros((sq, Hh, d), device=dev)
    kernels.set_algo("tc")
    kernels.attn_fwd_update(qq, kk, vv, m, l, acc, scale)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record()
    for _ in range(n):
        kernels.attn_fwd_update(qq, kk, vv, m, l, acc, scale)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 4.0 * sq * sk * d * Hh
    print(f"fwd block sq={sq} sk={sk} H={Hh}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")

# ---- backward: tcgen05 vs CUDA-core vs fp64 autograd ----
S2, H2 = int(os.environ.get("BS", "700")), 2
q2, k2, v2, do2 = (torch.randn(S2, H2, d, device=dev).to(torch.bfloat16) for _ in range(4))
qd, kd, vd = (t.double().requires_grad_() for t in (q2, k2, v2))
att = torch.softmax(torch.einsum("qhd,khd->hqk", qd, kd) * scale, -1)
od = torch.einsum("hqk,khd->qhd", att, vd)
od.backward(do2.double())


def bwd(algo):
    kernels.set_algo(algo)
    out, lse = run(algo, q2, k2, v2)
    delta = torch.empty((S2, H2), device=dev)
    kernels.attn_bwd_preprocess(out, do2, delta)
    dq = torch.zeros((S2, H2, d), device=dev)
    dk = torch.zeros_like(dq)
    dv = torch.zeros_like(dq)
    cuts = [0, S2 // 3, S2]
    for a, b in zip(cuts[:-1], cuts[1:]):
        kernels.attn_bwd_update(q2, k2[a:b], v2[a:b], do2, lse, delta, dq, dk[a:b], dv[a:b], scale)
    return dq, dk, dv


for algo in ("tc", "simt"):
    g = bwd(algo)
    errs = [((a.double() - b.grad).abs().max() / b.grad.abs().max()).item()
            for a, b in zip(g, (qd, kd, vd))]
    print(f"bwd {algo}: rel err dq {errs[0]:.3e} dk {errs[1]:.3e} dv {errs[2]:.3e}")

for (sq, sk) in ((8192, 8192), (65536, 65536)):
    Hh = 16
    qq, kk, vv, dd = (torch.randn(sq if i in (0, 3) else sk, Hh, d, device=dev).to(torch.bfloat16)
                      for i in range(4))
    lse = torch.randn(sq, Hh, device=dev) + 10
    delta = torch.randn(sq, Hh, device=dev)
    dq = torch.zeros((sq, Hh, d), device=dev)
    dk = torch.zeros((sk, Hh, d), device=dev)
    dv = torch.zeros_like(dk)
    kernels.set_algo("tc")
    kernels.attn_bwd_update(qq, kk, vv, dd, lse, delta, dq, dk, dv, scale)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 2
    e0.record()
    for _ in range(n):
        kernels.attn_bwd_update(qq, kk, vv, dd, lse, delta, dq, dk, dv, scale)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 2.5 * 4.0 * sq * sk * d * Hh
    print(f"bwd block sq={sq} sk={sk} H={Hh}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
