"""Host (Python + ctypes) cost of one cfg2 block step at the per-rank size of
an 8-GPU strong-scaling run (32 of 256 D-planes): is the GPU fed?

    python scripts/host_overhead.py [D]

Prints the device time per step (CUDA events), the host wall time per step
when steps are enqueued back to back (no sync), and a cProfile of the host
side."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_11111_b200 as dp  # noqa: E402

D = int(sys.argv[1]) if len(sys.argv) > 1 else 32
G, C0, C1 = 256, 16, 32


def prog(ctx):
    dev = ctx.device
    fmt = torch.channels_last_3d
    x = torch.randn((1, C0, D, G, G), device=dev, dtype=torch.bfloat16).contiguous(memory_format=fmt)
    w1 = (torch.randn((C1, C0, 3, 3, 3), device=dev) * 0.05).to(torch.bfloat16)
    w2 = (torch.randn((C1, C1, 3, 3, 3), device=dev) * 0.05).to(torch.bfloat16)
    xst = dp.ShardTensor(x, (1, C0, D, G, G), ctx, (dp.Shard(2),), {0: (D,)})
    g = torch.randn((1, C1, D, G, G), device=dev, dtype=torch.bfloat16).contiguous(memory_format=fmt)

    def step():
        y1, t1 = dp.halo_conv_forward(xst, w1, 1, 1)
        y2, t2 = dp.halo_conv_forward(y1, w2, 1, 1)
        dy1, dw2 = dp.halo_conv_backward(t2, g)
        dx, dw1 = dp.halo_conv_backward(t1, dy1)
        return dw1, dw2

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    n = 50
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    t_host = (time.perf_counter() - t0) / n
    e.record()
    torch.cuda.synchronize()
    t_dev = s.elapsed_time(e) / n
    print(f"D={D}: device {t_dev:.3f} ms/step (events, back to back), host enqueue "
          f"{1000 * t_host:.3f} ms/step, transport "
          f"{ctx.transport.kind}")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        step()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if os.environ.get("BACKEND", "thread") == "nccl":
    # one-process NCCL world: the NativeTransport the N-GPU runs use
    os.environ.setdefault("WORLD_SIZE", "1")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    prog(dp.init_mesh((1,), ("domain",)))
else:
    dp.spawn_mesh((1,), ("domain",), prog, device=torch.device("cuda", 0))
