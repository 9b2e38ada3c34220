"""Time the bf16x3 weight gradient over pre-split parts on the cfg1 grid
(DP_CONV_DBG ablations apply to the TS kernel: 1 no transpose, 2 no MMA, 4 no TMA)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels as k  # noqa: E402

G = int(os.environ.get("G", "1024"))
dev = torch.device("cuda", 0)
x = torch.randn((1, 32, G, G), device=dev)
dy = torch.randn((1, 32, G, G), device=dev)
dw = torch.empty((32, 32, 3, 3), device=dev)
kw = dict(kernel=(3, 3), stride=(1, 1), base=[-1, -1], shard=0, halo_rows=0)
g = k.conv_geom(x, None, dy.shape, dy.stride(), 32, (3, 3), (1, 1), [-1, -1], 0, 0)
xp = k.x3_split(x, k.X3_X, g)
dyp = k.x3_split(dy, k.X3_DY, g)
fn = lambda: k.conv_wgrad_x3(x, None, xp, None, dy, dyp, dw, **kw)  # noqa: E731
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
print(f"x3 wgrad parts G={G} dbg={os.environ.get('DP_CONV_DBG', '0')}: {ms:.4f} ms "
      f"{6 * 2.0 * 32 * 32 * 9 * G * G / ms / 1e9:.0f} bf16 TF/s")
