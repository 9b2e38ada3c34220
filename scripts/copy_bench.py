"""HBM roofline check of the data-movement kernels (dp_copy_strided /
dp_accumulate_strided) on the layouts the hot path moves: achieved GB/s =
(bytes read + bytes written) / CUDA-event time, vs MEASURED_PEAKS hbm_gbs."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_11111_b200 import kernels  # noqa: E402

dev = torch.device("cuda", 0)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def bench(name, fn, nbytes, n=20):
    """Device time per call: n calls captured in a CUDA graph and replayed
    (no host launch overhead between the kernels)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    gbs = nbytes / ms / 1e6
    print(f"{name:58s} {ms:8.3f} ms {gbs:8.1f} GB/s  {gbs / peak:5.1%} of {peak:.0f}")
    return gbs


out = {}
# contiguous 1 GiB fp32 (full_tensor / S->R slab landing)
a = torch.empty(256 * 2 ** 20, device=dev)
b = torch.empty_like(a)
out["contiguous_1GiB"] = bench("contiguous copy 1 GiB", lambda: kernels.copy_strided(b, a), 2 * a.numel() * 4)
# redistribute S(0)->S(1) pack: row slab [n/8, n] -> column block [n/8, n/8] x 8
n = 16384
slab = torch.empty((n // 8, n), device=dev)
packs = [torch.empty((n // 8, n // 8), device=dev) for _ in range(8)]


def pack_cols():
    for j in range(8):
        kernels.copy_strided(packs[j], slab[:, j * (n // 8):(j + 1) * (n // 8)])


out["redistribute_pack"] = bench("S(0)->S(1) column pack 128 MiB slab (8 blocks)", pack_cols,
                                 2 * slab.numel() * 4)
# W-sharded halo face pack: channels-last [1, 32, 64, 256, 256] bf16, last 2 W columns
x = torch.empty((1, 32, 64, 256, 256), device=dev, dtype=torch.bfloat16).contiguous(
    memory_format=torch.channels_last_3d)
face = torch.empty((1, 32, 64, 256, 2), device=dev, dtype=torch.bfloat16).contiguous(
    memory_format=torch.channels_last_3d)
out["halo_face_w"] = bench("halo face pack, W-sharded NDHWC bf16 (2 cols)",
                           lambda: kernels.copy_strided(face, x[..., -2:]), 2 * face.numel() * 2)
# D-sharded NCDHW (not channels-last) face: [1, 32, 2, 256, 256] from [1, 32, 64, 256, 256]
xn = torch.empty((1, 32, 64, 256, 256), device=dev, dtype=torch.bfloat16)
facen = torch.empty((1, 32, 2, 256, 256), device=dev, dtype=torch.bfloat16)
out["halo_face_d_ncdhw"] = bench("halo face pack, D-sharded NCDHW bf16 (2 planes)",
                                 lambda: kernels.copy_strided(facen, xn[:, :, -2:]),
                                 2 * facen.numel() * 2)
# reverse-halo accumulate fp32 dK/dV-sized (64 MiB)
acc = torch.empty(16 * 2 ** 20, device=dev)
inc = torch.empty_like(acc)
out["accumulate_64MiB"] = bench("accumulate 64 MiB fp32", lambda: kernels.accumulate(acc, inc),
                                3 * acc.numel() * 4)
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
