"""List every CUDA kernel smoke() launches (name -> count) with the torch
profiler, so eager-PyTorch kernels on the product path show up."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.smoke()   # warm (lazy module loads)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.smoke()
    torch.cuda.synchronize()
cnt = collections.Counter(e.name for e in prof.events() if e.device_type.name == "CUDA")
for name, n in sorted(cnt.items(), key=lambda kv: -kv[1]):
    print(f"{n:5d}  {name[:150]}")
