"""Time one tcgen05 conv launch on a cfg2-shaped volume (profiling helper).

    DP_CONV_DBG=<flags> python scripts/conv_time.py [fwd|dgrad|wgrad] [c_in] [c_out]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 32
co = int(sys.argv[3]) if len(sys.argv) > 3 else 32
G = int(os.environ.get("G", "256"))
dev = torch.device("cuda", 0)
cl = torch.channels_last_3d
x = torch.randn((1, ci, G, G, G), device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
w = (torch.randn((co, ci, 3, 3, 3), device=dev) * 0.05).to(torch.bfloat16)
# random dY too: zero operands draw less tensor-core power and run faster than
# the step's real activations
y = torch.randn((1, co, G, G, G), device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
dw = torch.empty((co, ci, 3, 3, 3), device=dev, dtype=torch.float32)
kw = dict(kernel=(3, 3, 3), stride=(1, 1, 1), base=[-1, -1, -1], shard=-1, halo_rows=0)


def run():
    if which == "fwd":
        kernels.conv_fwd(x, None, w, y, **kw)
    elif which == "dgrad":
        kernels.conv_dgrad(y, w, x, None, **kw)
    else:
        kernels.conv_wgrad(x, None, y, dw, **kw)


for _ in range(3):
    run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
s.record()
for _ in range(n):
    run()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
flops = 2.0 * ci * co * 27 * G ** 3
print(f"{which} ci={ci} co={co} dbg={os.environ.get('DP_CONV_DBG', '0')}: {ms:.3f} ms "
      f"{flops / ms / 1e9:.1f} TFLOP/s")
