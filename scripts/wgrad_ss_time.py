"""Time the SS weight gradient on cfg4's 64 -> 64 2-D layer (profiling helper);
the r4u sweep used temporary DP_WGRAD_KT / DP_WGRAD_SSNX planner knobs (not kept)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

G = int(os.environ.get("G", "2048"))
dev = torch.device("cuda", 0)
cl = torch.channels_last
x = torch.randn((1, 64, G, G), device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
dy = torch.randn((1, 64, G, G), device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
dw = torch.empty((64, 64, 3, 3), device=dev, dtype=torch.float32)
kw = dict(kernel=(3, 3), stride=(1, 1), base=[-1, -1], shard=-1, halo_rows=0)
fn = lambda: kernels.conv_wgrad(x, None, dy, dw, **kw)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    fn()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"ss wgrad 64->64 G={G} kt={os.environ.get('DP_WGRAD_KT', '-')} nx={os.environ.get('DP_WGRAD_SSNX', '-')}: "
      f"{ms:.4f} ms {2 * 64 * 64 * 9 * G * G / ms / 1e9:.1f} TFLOP/s")
