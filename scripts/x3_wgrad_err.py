"""dW error of the bf16x3 weight gradient on the full cfg1 grid vs an fp64
cuDNN reference, for the current DP_WGRAD_RF_ROWS (flush group)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels as k  # noqa: E402

G = 1024
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(101)
x = torch.randn((1, 32, G, G), device=dev, generator=gen)
dy = torch.randn((1, 32, G, G), device=dev, generator=gen)
dw = torch.empty((32, 32, 3, 3), device=dev)
kw = dict(kernel=(3, 3), stride=(1, 1), base=[-1, -1], shard=0, halo_rows=0)
g = k.conv_geom(x, None, dy.shape, dy.stride(), 32, (3, 3), (1, 1), [-1, -1], 0, 0)
xp, dyp = k.x3_split(x, k.X3_X, g), k.x3_split(dy, k.X3_DY, g)
k.conv_wgrad_x3(x, None, xp, None, dy, dyp, dw, **kw)
ref = torch.nn.grad.conv2d_weight(x.double(), (32, 32, 3, 3), dy.double(), padding=1)
err = ((dw.double() - ref).abs().max() / ref.abs().max()).item()
print(f"rf_rows={os.environ.get('DP_WGRAD_RF_ROWS', 'default')}: dW rel err {err:.2e}")
