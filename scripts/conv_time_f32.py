"""Time the fp32 CUDA-core conv kernels on the cfg1 grid (1x32x1024x1024, 3x3)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11111_b200 import kernels  # noqa: E402

G = int(os.environ.get("G", "1024"))
dev = torch.device("cuda", 0)
x = torch.randn((1, 32, G, G), device=dev)
w = torch.randn((32, 32, 3, 3), device=dev) * 0.05
y = torch.empty((1, 32, G, G), device=dev)
dw = torch.empty((32, 32, 3, 3), device=dev)
kw = dict(kernel=(3, 3), stride=(1, 1), base=[-1, -1], shard=-1, halo_rows=0)
fl = 2.0 * 32 * 32 * 9 * G * G
for name, fn in (("fwd", lambda: kernels.conv_fwd(x, None, w, y, **kw)),
                 ("dgrad", lambda: kernels.conv_dgrad(y, w, x, None, **kw)),
                 ("wgrad", lambda: kernels.conv_wgrad(x, None, y, dw, **kw))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{name} f32: {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s")
