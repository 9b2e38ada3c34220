#!/usr/bin/env python
"""Benchmark of the B200 domain-parallel hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Default workload = BASELINE.json configs[1] (cfg2): the UNet-style conv3d
encoder block conv(16->32, 3^3) -> conv(32->32, 3^3), stride 1, padding 1,
no bias/activation (the reference conv has neither), on a 1x16x256^3 bf16
volume D-sharded over N GPUs (strong scaling).  One step = forward of both
layers + backward (dgrad of both layers incl. the block input, wgrad of
both, reverse halos, dW all-reduce) against a fixed synthetic upstream
gradient.  Activations live channels-last (NDHWC) in HBM.

Other configs (--config): cfg1 (conv2d fp32 parity anchor, R=2 semantics on
N GPUs), cfg3 (ring attention 64k x 16 heads x 64, bf16), cfg4 (weak-scaling
conv2d stack 64ch x4 on 2048^2 per GPU), cfg5 (uneven redistribute).

Rank 0 prints ONE JSON line.  `value` = samples/s of the whole job with
inputs resident in HBM (device time, CUDA events, max over ranks); `e2e` =
the same through the public API with the input shard copied host->device
(pinned) and dW read back device->host every step; `roofline` = the
dominant kernel's achieved TFLOP/s (algorithmic FLOPs / measured launch
time) vs the measured bf16 peak in MEASURED_PEAKS.json; `cpu_baseline` =
the oracle port of the reference algorithm timed on a bounded sample on
this host.  `--impl reference` times that CPU implementation as the
reference arm (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


SIZE_MIB = 1024   # cfg5 tensor size (--size-mib)

# workload names shared by both arms (ours and --impl reference)
WORKLOAD_TEXT = {
    "cfg2": "cfg2: conv3d 3x3x3 UNet-style encoder block conv(16->32)->conv(32->32), s1 p1, "
            "no bias/activation, 1x16x256^3 bf16, D-sharded",
    "cfg3": "cfg3: ring-attention SDPA, ViT-style 64k-token sequence, 16 heads, d=64, bf16, "
            "non-causal, scale 1/8, sequence-sharded",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--algo", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--size-mib", type=int, default=1024,
                    help="cfg5: global tensor size (the sweep runs 64 .. 8192)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    """SM clock + clock-event reasons sampled through NVML every 10 ms while
    the timed region runs (best effort: no NVML -> no samples)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []   # (sm_mhz, reasons bitmask)
        self.power = []     # board power draw, W
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def _handle(self):
        import pynvml

        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.gpu
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.gpu < len(ids) and ids[self.gpu].isdigit():
                idx = int(ids[self.gpu])
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _run(self):
        nv, h = self._nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                              getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = get_reasons(h) if get_reasons else 0
                self.samples.append((sm, rs))
                self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)   # W
            except Exception:  # noqa: BLE001 - sampling is best effort
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        try:
            self._nvml = self._handle()
            nv, h = self._nvml
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self._nvml = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        nv = self._nvml[0]
        reasons = set()
        for _, rs in self.samples:
            for name, attr in self.REASONS:
                bit = getattr(nv, attr, 0)
                if bit and rs & bit:
                    reasons.add(name)
        sms = sorted(sm for sm, _ in self.samples)
        out = {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": self.max_mhz,
               "sm_min_mhz": sms[0], "reasons": sorted(reasons), "samples": len(sms),
               "source": "nvml 10 ms"}
        if self.power:
            pw = sorted(self.power)
            out.update({"power_w_median": pw[len(pw) // 2], "power_w_max": pw[-1]})
            try:
                nv, h = self._nvml
                out["power_limit_w"] = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
            except Exception:  # noqa: BLE001
                pass
        return out


# ---------------------------------------------------------------------------
# mesh


def init(args):
    import torch

    import paper_2605_11111_b200 as dp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world == 1 and "MASTER_PORT" not in os.environ:
        import socket

        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(s.getsockname()[1])
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    ctx = dp.init_mesh((world,), ("domain",))
    torch.cuda.set_device(ctx.device)
    return ctx


def max_over_ranks(ctx, value: float) -> float:
    import torch
    import torch.distributed as dist

    if ctx.mesh.world_size == 1:
        return value
    dev = ctx.device if dist.get_backend() == "nccl" else "cpu"   # gloo dry runs: host
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ctx):
    import torch
    import torch.distributed as dist

    if ctx.mesh.world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# kernel-level timing INSIDE the timed region: CUDA events around every conv /
# attention call, recorded on the stream the call launches on (the current
# stream), keyed by entry point and layer shape


class KernelTimer:
    NAMES = ("conv_fwd", "conv_dgrad", "conv_wgrad", "attn_fwd_update", "attn_bwd_update",
             "conv_fwd_x3", "conv_dgrad_x3", "conv_wgrad_x3", "x3_split")

    def __init__(self):
        self.records = []  # (key, flops, start, end)
        self.active = False

    def wrap(self, kernels_mod):
        import torch

        timer = self
        for name in self.NAMES:
            orig = getattr(kernels_mod, name)

            def make(orig=orig, name=name):
                def inner(*a, **kw):
                    if not timer.active:
                        return orig(*a, **kw)
                    flops, tag = kernel_work(name, a, kw)
                    s = torch.cuda.Event(enable_timing=True)
                    e = torch.cuda.Event(enable_timing=True)
                    s.record()
                    res = orig(*a, **kw)
                    e.record()
                    base = name.replace("_x3", "")
                    nbytes = 0
                    if name == "x3_split":   # fp32 read + 3 bf16 parts written (HBM-bound)
                        nbytes = a[0].numel() * (4 + 3 * 2)
                    timer.records.append((f"{base}[{tag}]", flops, s, e, nbytes))
                    return res
                return inner
            setattr(kernels_mod, name, make())

    def summary(self):
        import torch

        torch.cuda.synchronize()
        out = {}
        for key, flops, s, e, nbytes in self.records:
            d = out.setdefault(key, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0})
            d["launches"] += 1
            d["ms"] += s.elapsed_time(e)
            d["flops"] += flops
            d["bytes"] += nbytes
        return out


class CommMeter:
    """Bytes this rank posts to its peers (every send of every exchange round)
    while active: halo faces, reverse halos, K||V hops, redistribute blocks,
    all-reduce payloads."""

    def __init__(self):
        self.bytes = 0
        self.calls = 0
        self.active = False

    def wrap(self, transport):
        meter = self
        orig_start = transport.exchange_start
        orig_ex = transport.exchange
        orig_ar = transport.all_reduce

        def count(sends):
            if meter.active:
                meter.calls += 1
                meter.bytes += sum(t.numel() * t.element_size() for _, t in sends)

        def exchange_start(sends, recvs):
            count(sends)
            return orig_start(sends, recvs)

        def exchange(sends, recvs):
            count(sends)
            return orig_ex(sends, recvs)

        def all_reduce(members, me, t, op):
            if meter.active:
                meter.calls += 1
                meter.bytes += t.numel() * t.element_size() * (len(members) - 1)
            return orig_ar(members, me, t, op)

        # the thread mailbox's exchange_start calls exchange; the process
        # transports' exchange calls exchange_start: wrap the inner one only
        if getattr(transport, "kind", "") == "thread":
            transport.exchange = exchange
        else:
            transport.exchange_start = exchange_start
        transport.all_reduce = all_reduce


def kernel_work(name, a, kw):
    """Algorithmic work of one wrapped call: FLOPs for conv / attention
    (conv: 2 * C_in * C_out * taps * output positions of the forward conv it
    belongs to — dgrad and wgrad count the same MACs; attention fwd block:
    4 * sq * sk * d * H; bwd block: 2.5x that, the 5-GEMM convention of
    SURVEY 8(d))."""
    import math

    if name == "x3_split":       # bf16x3 operand split: data movement, no FLOPs
        return 0.0, "fp32->3xbf16"
    if name == "conv_fwd":
        x, _, w, y = a[:4]
        pos = y.shape[0] * math.prod(y.shape[2:])
    elif name == "conv_fwd_x3":      # (x, x_halo, xp, xhp, w, y)
        w, y = a[4], a[5]
        pos = y.shape[0] * math.prod(y.shape[2:])
    elif name == "conv_dgrad":
        dy, w = a[0], a[1]
        pos = dy.shape[0] * math.prod(dy.shape[2:])
    elif name == "conv_dgrad_x3":    # (dy, dyp, w, dx, dx_halo)
        dy, w = a[0], a[2]
        pos = dy.shape[0] * math.prod(dy.shape[2:])
    elif name == "conv_wgrad_x3":    # (x, x_halo, xp, xhp, dy, dyp, dw)
        dy, w = a[4], a[6]
        pos = dy.shape[0] * math.prod(dy.shape[2:])
    elif name == "conv_wgrad":
        x, _, dy, w = a[0], a[1], a[2], a[3]
        pos = dy.shape[0] * math.prod(dy.shape[2:])
    else:  # attention blocks
        q, k = a[0], a[1]
        heads = q.shape[1] if q.dim() == 3 else 1
        f = 4.0 * q.shape[0] * k.shape[0] * q.shape[-1] * heads
        return f * (2.5 if name == "attn_bwd_update" else 1.0), f"d{q.shape[-1]}"
    tag = f"{w.shape[1]}->{w.shape[0]}"   # layer: c_in -> c_out (same for fwd, dgrad, wgrad)
    return 2.0 * w.shape[0] * w.shape[1] * math.prod(w.shape[2:]) * pos, tag


# ---------------------------------------------------------------------------
# workloads (ours)


def cfg5_n() -> int:
    return int(round((SIZE_MIB * 2 ** 20 / 4) ** 0.5)) // 8 * 8   # [n, n] fp32


def workload_info(name: str, R: int) -> dict:
    """The `config` object of the JSON line — built from the config name and
    the rank count only, so both arms (ours and --impl reference) print the
    identical object."""
    from paper_2605_11111_b200.plan import default_chunk

    if name == "cfg2":
        return {"workload": WORKLOAD_TEXT["cfg2"], "global_batch": 1, "volume": [256] * 3,
                "channels": [16, 32, 32], "layout": "NDHWC (channels_last_3d)",
                "shard_extents": list(default_chunk(256, R)), "parallelism": f"domain{R}",
                "l2": "inputs larger than L2 (512 MiB activations per layer), no flush"}
    if name == "cfg3":
        return {"workload": WORKLOAD_TEXT["cfg3"], "global_batch": 1, "seq_len": 65536,
                "heads": 16, "head_dim": 64, "shard_extents": list(default_chunk(65536, R)),
                "parallelism": f"ring{R}",
                "l2": "inputs (q, k, v, dO: 512 MiB) exceed L2, no flush"}
    if name == "cfg4":
        return {"workload": "cfg4: weak-scaling conv2d stack, 4 x conv(64->64, 3x3, s1 p1), "
                            "2048^2 per GPU, bf16, H-sharded",
                "global_batch": 1, "grid_per_gpu": [2048, 2048], "channels": 64, "layers": 4,
                "layout": "NHWC (channels_last)", "shard_extents": [2048] * R,
                "parallelism": f"domain{R}",
                "l2": "inputs larger than L2 (512 MiB activations per layer), no flush"}
    if name == "cfg5":
        n = cfg5_n()
        return {"workload": f"cfg5: uneven redistribute of a [{n},{n}] fp32 tensor "
                            f"({n * n * 4 / 2 ** 20:.0f} MiB), Shard(0) random_partition extents "
                            "-> Replicate and -> Shard(1)",
                "global_batch": 1, "shape": [n, n], "shard_extents": random_partition(R, n, R),
                "parallelism": f"domain{R}", "l2": "tensor exceeds L2, no flush"}
    return {"workload": "cfg1: conv2d 3x3 halo exchange, 1x32x1024x1024 fp32, C_out=32, s1 p1, "
                        "H-sharded (fp32 on the tensor cores as exact bf16x3 part products: the "
                        "reference's 1e-5 tolerance)",
            "global_batch": 1, "grid": [1024, 1024], "channels": [32, 32], "layout": "NCHW",
            "shard_extents": list(default_chunk(1024, R)), "parallelism": f"domain{R}",
            "l2": "128 MiB activations exceed L2, no flush"}


def setup_cfg2(ctx):
    import torch

    import paper_2605_11111_b200 as dp

    G, C0, C1 = 256, 16, 32
    R = ctx.mesh.world_size
    me = ctx.rank_id
    dev = ctx.device
    ext = dp.default_chunk(G, R)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + me)
    fmt = torch.channels_last_3d
    x = torch.randn((1, C0, ext[me], G, G), generator=gen, device=dev, dtype=torch.bfloat16)
    x = x.contiguous(memory_format=fmt)
    wg = torch.Generator(device=dev)
    wg.manual_seed(7)  # identical weights on every rank (replicated)
    w1 = (torch.randn((C1, C0, 3, 3, 3), generator=wg, device=dev) * 0.05).to(torch.bfloat16)
    w2 = (torch.randn((C1, C1, 3, 3, 3), generator=wg, device=dev) * 0.05).to(torch.bfloat16)
    p1 = dp.halo_conv_plan(ext, G, 3, 1, 1)
    p2 = dp.halo_conv_plan(list(p1.out_extents), G, 3, 1, 1)
    g = torch.randn((1, C1, p2.out_extents[me], G, G), generator=gen, device=dev,
                    dtype=torch.bfloat16).contiguous(memory_format=fmt)
    xst = dp.ShardTensor(x, (1, C0, G, G, G), ctx, (dp.Shard(2),), {0: tuple(ext)})

    def step(ins=None):
        st = xst if ins is None else dp.ShardTensor(ins[0], xst.global_shape, ctx, xst.placements,
                                                    xst.shard_shapes)
        y1, t1 = dp.halo_conv_forward(st, w1, 1, 1)
        y2, t2 = dp.halo_conv_forward(y1, w2, 1, 1)
        dy1, dw2 = dp.halo_conv_backward(t2, g)
        dx, dw1 = dp.halo_conv_backward(t1, dy1)
        return dw1, dw2

    flops = 3 * 2.0 * (C0 * C1 + C1 * C1) * 27 * G ** 3  # fwd + dgrad + wgrad, both layers
    info = workload_info("cfg2", R)
    return dict(step=step, inputs=[x], flops=flops, info=info, scaling="strong", dtype="bf16",
                unit="samples/s", samples_per_step=1)


def cpu_sample_cfg2(threads: int):
    """Oracle port of the reference algorithm on a bounded sample: the
    block fwd+bwd on `threads` independent sub-volumes of 1 x 256 x 64
    voxels (each 1/1024 of the volume), fp32, one per thread.  Returns
    (seconds, fraction of one sample computed)."""
    import numpy as np

    from oracle import workloads

    rng = np.random.default_rng(0)
    w1 = (rng.standard_normal((32, 16, 3, 3, 3)) * 0.05).astype(np.float32)
    w2 = (rng.standard_normal((32, 32, 3, 3, 3)) * 0.05).astype(np.float32)
    jobs = []
    for _ in range(threads):
        x = rng.standard_normal((1, 16, 1, 256, 64)).astype(np.float32)
        g = rng.standard_normal((1, 32, 1, 256, 64)).astype(np.float32)
        jobs.append((x, g))
    t0 = time.perf_counter()
    if threads == 1:
        workloads.conv_block_step(jobs[0][0], w1, w2, jobs[0][1])
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda j: workloads.conv_block_step(j[0], w1, w2, j[1]), jobs))
    dt = time.perf_counter() - t0
    return dt, threads / 1024.0


def setup_cfg3(ctx):
    """Ring attention, ViT-style 64k-token sequence, 16 heads, d = 64, bf16,
    sequence-sharded (Shard(0), default_chunk) over the N ranks.  One step =
    ring_attention forward + backward (R-1 K||V hops forward, R (K,V,dK,dV)
    hops backward) against a fixed synthetic dO."""
    import torch

    import paper_2605_11111_b200 as dp

    S, H, D = 65536, 16, 64
    R = ctx.mesh.world_size
    me = ctx.rank_id
    dev = ctx.device
    ext = dp.default_chunk(S, R)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + me)
    q, k, v, do = (torch.randn((ext[me], H, D), generator=gen, device=dev,
                               dtype=torch.bfloat16) for _ in range(4))
    shards = {0: tuple(ext)}
    kst = dp.ShardTensor(k, (S, H, D), ctx, (dp.Shard(0),), shards)
    vst = dp.ShardTensor(v, (S, H, D), ctx, (dp.Shard(0),), shards)
    qst = dp.ShardTensor(q, (S, H, D), ctx, (dp.Shard(0),), shards)

    def step(ins=None):
        if ins is None:
            qs, ks, vs, g = qst, kst, vst, do
        else:
            qs, ks, vs = (dp.ShardTensor(t, (S, H, D), ctx, (dp.Shard(0),), shards)
                          for t in ins[:3])
            g = ins[3]
        out, tape = dp.ring_attention_forward(qs, ks, vs)
        dq, dk, dv = dp.ring_attention_backward(tape, g)
        return dq.local, dk.local, dv.local

    flops = 3.5 * 4.0 * S * S * D * H  # fwd + 2.5x bwd
    info = workload_info("cfg3", R)
    return dict(step=step, inputs=[q, k, v, do], flops=flops, info=info, scaling="strong",
                dtype="bf16", unit="samples/s", samples_per_step=1)


def cpu_sample_cfg3(threads: int):
    """Oracle port on a bounded sample: per thread one head's 128 query rows
    against all 65536 keys, fwd + bwd in fp64 softmax (1/8192 of the cfg3
    fwd+bwd work each)."""
    import numpy as np

    from oracle import workloads

    rng = np.random.default_rng(0)
    S, D, rows = 65536, 64, 128
    k = rng.standard_normal((S, D)).astype(np.float32)
    v = rng.standard_normal((S, D)).astype(np.float32)
    jobs = [(rng.standard_normal((rows, D)).astype(np.float32),
             rng.standard_normal((rows, D)).astype(np.float32)) for _ in range(threads)]
    t0 = time.perf_counter()
    if threads == 1:
        workloads.attention_step(jobs[0][0], k, v, jobs[0][1])
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda j: workloads.attention_step(j[0], k, v, j[1]), jobs))
    dt = time.perf_counter() - t0
    return dt, threads * rows / (S * 16.0)


def setup_cfg4(ctx):
    """Weak-scaling 2-D conv stack: 4 x conv(64->64, 3x3, s1, p1), 2048^2
    per GPU (global [1, 64, 2048*R, 2048], Shard(2)), bf16 NHWC.  One step
    = forward of the 4 layers + backward (dgrad incl. the stack input,
    wgrad, reverse halos, dW all-reduces)."""
    import torch

    import paper_2605_11111_b200 as dp

    C, L, Hper, W = 64, 4, 2048, 2048
    R = ctx.mesh.world_size
    me = ctx.rank_id
    dev = ctx.device
    G = Hper * R
    ext = [Hper] * R
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + me)
    fmt = torch.channels_last
    x = torch.randn((1, C, Hper, W), generator=gen, device=dev,
                    dtype=torch.bfloat16).contiguous(memory_format=fmt)
    wg = torch.Generator(device=dev)
    wg.manual_seed(11)
    ws = [(torch.randn((C, C, 3, 3), generator=wg, device=dev) * 0.05).to(torch.bfloat16)
          for _ in range(L)]
    plans = []
    cur = ext
    for _ in range(L):
        pl = dp.halo_conv_plan(cur, G, 3, 1, 1)
        plans.append(pl)
        cur = list(pl.out_extents)
    g = torch.randn((1, C, cur[me], W), generator=gen, device=dev,
                    dtype=torch.bfloat16).contiguous(memory_format=fmt)
    xst = dp.ShardTensor(x, (1, C, G, W), ctx, (dp.Shard(2),), {0: tuple(ext)})

    def step(ins=None):
        st = xst if ins is None else dp.ShardTensor(ins[0], xst.global_shape, ctx, xst.placements,
                                                    xst.shard_shapes)
        tapes = []
        for w in ws:
            st, t = dp.halo_conv_forward(st, w, 1, 1)
            tapes.append(t)
        dy = g
        dws = []
        for t in reversed(tapes):
            dxs, dw = dp.halo_conv_backward(t, dy)
            dy = dxs.local
            dws.append(dw)
        return dws

    flops = 3 * L * 2.0 * C * C * 9 * Hper * W
    info = workload_info("cfg4", R)
    return dict(step=step, inputs=[x], flops=flops, info=info, scaling="weak", dtype="bf16",
                unit="samples/s", samples_per_step=1)


def cpu_sample_cfg4(threads: int):
    """Oracle port on a bounded sample: per thread a 1 x 64 x 16 x 256 tile
    through the 4-layer stack fwd+bwd (1/1024 of one GPU's 2048^2 step)."""
    import numpy as np

    from oracle import workloads

    rng = np.random.default_rng(0)
    ws = [(rng.standard_normal((64, 64, 3, 3)) * 0.05).astype(np.float32) for _ in range(4)]
    jobs = [(rng.standard_normal((1, 64, 16, 256)).astype(np.float32),
             rng.standard_normal((1, 64, 16, 256)).astype(np.float32)) for _ in range(threads)]
    t0 = time.perf_counter()
    if threads == 1:
        workloads.conv_stack_step(jobs[0][0], ws, jobs[0][1])
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda j: workloads.conv_stack_step(j[0], ws, j[1]), jobs))
    dt = time.perf_counter() - t0
    return dt, threads / 1024.0



def random_partition(seed: int, n: int, parts: int, min_part: int = 1):
    """Uneven extents exactly as the reference's workload generator
    (domainpar/verify.py:67-81) with rng = default_rng(seed)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    if parts == 1:
        return [n]
    spare = n - min_part * parts
    cuts = np.sort(rng.integers(0, spare + 1, size=parts - 1))
    edges = [0, *cuts.tolist(), spare]
    return [min_part + edges[i + 1] - edges[i] for i in range(parts)]


def setup_cfg5(ctx):
    """Uneven-shard redistribute: a [n, n] fp32 tensor (1 GiB) Shard(0) with
    random_partition extents -> Replicate (varlen all-gather) and -> Shard(1)
    (variable-count all-to-all).  One step = both redistributions."""
    import torch

    import paper_2605_11111_b200 as dp

    n = cfg5_n()
    R = ctx.mesh.world_size
    me = ctx.rank_id
    dev = ctx.device
    ext = random_partition(R, n, R)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5 + me)
    local = torch.randn((ext[me], n), generator=gen, device=dev)
    st = dp.ShardTensor(local, (n, n), ctx, (dp.Shard(0),), {0: tuple(ext)})

    def step(ins=None):
        s0 = st if ins is None else dp.ShardTensor(ins[0], (n, n), ctx, (dp.Shard(0),),
                                                   {0: tuple(ext)})
        rep = dp.redistribute(s0, (dp.Replicate(),))
        s1 = dp.redistribute(s0, (dp.Shard(1),))
        return rep.local[:1], s1.local[:1]

    info = workload_info("cfg5", R)
    # algorithmic HBM bytes of this rank's step: read its input block once and
    # write each output once (S(0) -> R: the whole [n, n]; S(0) -> S(1): [n, n/R])
    cshare = dp.default_chunk(n, R)[me]
    hbm = (ext[me] * n + n * n) * 4 + (ext[me] * n + n * cshare) * 4
    extra = {"bytes_received_per_rank": {"to_replicate": (n - ext[me]) * n * 4,
                                         "to_shard1": (n - ext[me]) * cshare * 4},
             "hbm_bytes_per_step": hbm}
    return dict(step=step, inputs=[local], flops=0.0, info=info, scaling="strong", dtype="f32",
                hbm_bytes_per_step=hbm, extra=extra, unit="samples/s", samples_per_step=1)


def cpu_sample_cfg5(threads: int):
    """Oracle port on a bounded sample: the reference's gather-then-slice
    (np.concatenate + column slice) of a [4096, 16384] fp32 slab set (1/4 of
    the rows), `threads` rank threads."""
    import numpy as np

    from oracle import sharding as osh

    n, rows = 16384, 4096
    R = max(2, threads)
    ext = random_partition(R, rows, R)
    rng = np.random.default_rng(0)
    g = rng.standard_normal((rows, n)).astype(np.float32)
    b = np.concatenate([[0], np.cumsum(ext)])
    blocks = [g[b[i]:b[i + 1]] for i in range(R)]
    t0 = time.perf_counter()
    full = np.concatenate(blocks, axis=0)          # S(0) -> Replicate on every rank
    cols = osh.default_chunk(n, R)
    cb = np.concatenate([[0], np.cumsum(cols)])
    for i in range(R):                             # S(0) -> S(1): slice own columns
        np.ascontiguousarray(full[:, cb[i]:cb[i + 1]])
    dt = time.perf_counter() - t0
    return dt, rows / n


def setup_cfg1(ctx):
    """conv2d 3x3 halo exchange on a 1x32x1024x1024 fp32 grid, C_out = 32,
    s1 p1, H-sharded (the reference's CPU parity anchor; fp32 keeps the
    reference's 1e-5 tolerance, so it runs the fp32 CUDA-core kernels).
    One step = forward + backward."""
    import torch

    import paper_2605_11111_b200 as dp

    G, C = 1024, 32
    R = ctx.mesh.world_size
    me = ctx.rank_id
    dev = ctx.device
    ext = dp.default_chunk(G, R)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0 + me)
    x = torch.randn((1, C, ext[me], G), generator=gen, device=dev)
    wg = torch.Generator(device=dev)
    wg.manual_seed(1)
    w = torch.randn((C, C, 3, 3), generator=wg, device=dev) * 0.1
    plan = dp.halo_conv_plan(ext, G, 3, 1, 1)
    g = torch.randn((1, C, plan.out_extents[me], G), generator=gen, device=dev)
    xst = dp.ShardTensor(x, (1, C, G, G), ctx, (dp.Shard(2),), {0: tuple(ext)})

    def step(ins=None):
        st = xst if ins is None else dp.ShardTensor(ins[0], xst.global_shape, ctx, xst.placements,
                                                    xst.shard_shapes)
        y, t = dp.halo_conv_forward(st, w, 1, 1)
        dx, dw = dp.halo_conv_backward(t, g)
        return [dw]

    flops = 3 * 2.0 * C * C * 9 * G * G
    info = workload_info("cfg1", R)
    return dict(step=step, inputs=[x], flops=flops, info=info, scaling="strong", dtype="f32",
                unit="samples/s", samples_per_step=1)


def cpu_sample_cfg1(threads: int):
    """Oracle port (the reference's dense.conv einsum) on 1x32x16x1024
    row slabs, fwd+bwd, one per thread (1/64 of the grid each)."""
    import numpy as np

    from oracle import workloads

    rng = np.random.default_rng(0)
    w = (rng.standard_normal((32, 32, 3, 3)) * 0.1).astype(np.float32)
    jobs = [(rng.standard_normal((1, 32, 16, 1024)).astype(np.float32),
             rng.standard_normal((1, 32, 16, 1024)).astype(np.float32)) for _ in range(threads)]
    t0 = time.perf_counter()
    if threads == 1:
        workloads.conv_stack_step(jobs[0][0], [w], jobs[0][1])
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda j: workloads.conv_stack_step(j[0], [w], j[1]), jobs))
    dt = time.perf_counter() - t0
    return dt, threads / 64.0

CONFIGS = {"cfg2": (setup_cfg2, cpu_sample_cfg2,
                    "1 x 256 x 64 voxel sub-volumes (1/1024 of the 256^3 volume each), fp32, "
                    "block fwd+bwd via the oracle port of dense.conv's einsum"),
           "cfg3": (setup_cfg3, cpu_sample_cfg3,
                    "one head's 128 query rows vs all 65536 keys (1/8192 of the cfg3 step), "
                    "fp32 in / fp64 softmax, fwd+bwd via the oracle port"),
           "cfg1": (setup_cfg1, cpu_sample_cfg1,
                    "1 x 32 x 16 x 1024 fp32 row slabs (1/64 of the grid each), conv fwd+bwd via "
                    "the oracle port of dense.conv's einsum"),
           "cfg5": (setup_cfg5, cpu_sample_cfg5,
                    "np.concatenate + column slices of a 4096 x 16384 fp32 slab set (1/4 of the "
                    "rows), the reference's gather-then-slice"),
           "cfg4": (setup_cfg4, cpu_sample_cfg4,
                    "1 x 64 x 16 x 256 tiles (1/1024 of one GPU's 2048^2 stack step), fp32, "
                    "4-layer fwd+bwd via the oracle port")}


# ---------------------------------------------------------------------------


def run_reference(args):
    """The reference arm: the reference algorithm's CPU implementation (the
    oracle port of domainpar's NumPy path — the reference is Python and does
    not travel to this box) on all host threads.  Exactly W warm-up and K
    timed steps, each one bounded sample of the configured workload (the
    sample is named in cpu_baseline.sample); `value` = samples/s extrapolated
    from the sampled fraction, `ms_per_step` = the measured wall time of one
    sampled step, so K x ms_per_step is what this run actually spent."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    _, cpu_fn, sample_desc = CONFIGS[args.config]
    for _ in range(max(0, args.warmup)):
        cpu_fn(cores)
    times = []
    frac = 1.0
    for _ in range(max(1, args.steps)):
        dt, frac = cpu_fn(cores)
        times.append(dt)
    t = sum(times) / len(times)
    value = frac / t  # samples per second
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": len(times), "warmup": max(0, args.warmup),
            "ms_per_step": 1000.0 * t, "higher_is_better": True,
            "scaling": "weak" if args.config == "cfg4" else "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": workload_info(args.config, max(1, args.gpus)),
            "sample_fraction": frac,
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores,
                             "kind": "port", "sample": f"{cores} x {sample_desc}",
                             "sample_fraction_per_step": frac,
                             "note": "ms_per_step is one sampled step; value extrapolates "
                                     "samples/s from the sampled fraction"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "sharded fwd+bwd step latency & samples/s"


def self_launch(args) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks of this
    script the way torchrun would (RANK / LOCAL_RANK / WORLD_SIZE /
    MASTER_ADDR=127.0.0.1 / MASTER_PORT), one process per GPU over NCCL.
    With fewer visible GPUs than N (a one-GPU box) the ranks share the GPU
    over gloo ("gloo-cuda": the same one-process-per-rank code path, payloads
    staged through host memory) and the line says so."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    try:
        import torch

        ngpu = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        ngpu = 0
    base = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                WORLD_SIZE=str(args.gpus), LOCAL_WORLD_SIZE=str(args.gpus))
    if ngpu < args.gpus:
        base["DP_MESH_BACKEND"] = "gloo-cuda"
    procs = []
    for r in range(args.gpus):
        env = dict(base, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(abs(rc) for rc in rcs)


def pick_peak(pk, clk_summary, dtype):
    """Burst bf16 peak when the SM clock held (median >= 95 % of max) during
    the timed region, else the sustained one; fp32 runs on the tensor cores
    as six bf16 part products (conv_x3), so its roof is that / 6."""
    sm, mx = clk_summary.get("sm_mhz"), clk_summary.get("sm_max_mhz")
    burst = sm is None or mx is None or sm >= 0.95 * mx
    key = "bf16_tflops" if burst else "bf16_tflops_sustained"
    peak = pk.get(key, PEAKS_FALLBACK[key])
    kind = f"bf16 {'burst' if burst else 'sustained'} (SM clock median {sm} of {mx} MHz)"
    if dtype == "f32":
        peak /= 6.0
        kind += " / 6: fp32 = 6 bf16 part products on the tensor cores (conv_x3)"
    return peak, kind


def main():
    args = parse()
    global SIZE_MIB
    SIZE_MIB = args.size_mib
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(self_launch(args))
    import torch

    from paper_2605_11111_b200 import _lib, kernels

    kernels.set_algo(args.algo)
    ctx = init(args)
    _OPEN.append(ctx)
    setup_fn, cpu_fn, sample_desc = CONFIGS[args.config]
    W = setup_fn(ctx)
    step = W["step"]
    for _ in range(max(3, args.warmup)):
        step()
    timer = KernelTimer()
    timer.wrap(kernels)
    comm = CommMeter()
    comm.wrap(ctx.transport)
    barrier(ctx)

    # --- timed region: device time, inputs resident in HBM; every conv /
    # attention launch bracketed by CUDA events on its stream ----------------
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    l0, s0 = _lib.launch_count(), _lib.simt_count()
    local_gpu = ctx.device.index if ctx.device.index is not None else 0
    with ClockSampler(local_gpu) as clk:
        barrier(ctx)
        timer.active = comm.active = True
        if hasattr(ctx.transport, "timing"):
            ctx.transport.timing = []   # NativeTransport: events around every NCCL round
        start.record()
        for _ in range(args.steps):
            step()
        end.record()
        timer.active = comm.active = False
        barrier(ctx)
    launches = _lib.launch_count() - l0
    simt_calls = _lib.simt_count() - s0
    my_ms = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ctx, my_ms)
    ksum = timer.summary()
    comm_bytes = comm.bytes / args.steps
    nccl_ms = nccl_bytes = None
    if getattr(ctx.transport, "timing", None) is not None:
        rounds = ctx.transport.timing
        ctx.transport.timing = None
        nccl_ms = sum(a.elapsed_time(b) for a, b, _ in rounds) / args.steps
        nccl_bytes = sum(n for _, _, n in rounds) / args.steps
    kernel_ms_step = sum(v["ms"] for v in ksum.values()) / args.steps
    # every rank's per-kernel record (max over ranks for the roofline)
    ranks_k = gather_all(ctx, {"ksum": ksum, "ms": my_ms, "kernel_ms": kernel_ms_step,
                               "comm_bytes": comm_bytes, "simt": simt_calls,
                               "nccl_ms": nccl_ms, "nccl_bytes": nccl_bytes})

    # --- e2e through the public API: pinned host input -> device, gradients ->
    # host.  Every step copies its own input shard from pinned host memory and
    # reads its result back; the copy for step i+1 runs on a copy stream while
    # step i computes (double-buffered input, as a training loop's prefetcher
    # would), and step i's result drains to host on a third stream while step
    # i+1 computes (PCIe is full duplex: the H2D prefetch and the D2H drain run
    # at once), so the timed region = first H2D + K steps + last D2H.
    ins = W["inputs"]
    hosts = []
    for t in ins:
        h = torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        hosts.append(h)
    bufs = [[torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, device=t.device)
             for t in ins] for _ in range(2)]
    outs = step()
    host_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
    d2h = sum(o.numel() * o.element_size() for o in outs)
    h2d = sum(t.numel() * t.element_size() for t in ins)
    copy_stream = torch.cuda.Stream(device=ctx.device)
    d2h_stream = torch.cuda.Stream(device=ctx.device)
    compute = torch.cuda.current_stream()
    e2e_steps = max(1, args.steps)
    barrier(ctx)
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def upload(slot):
        for dst, src in zip(bufs[slot], hosts):
            dst.copy_(src, non_blocking=True)

    e_start.record(compute)
    with torch.cuda.stream(copy_stream):
        copy_stream.wait_event(e_start)
        upload(0)
        ready[0].record(copy_stream)
    for i in range(e2e_steps):
        cur = i % 2
        if i + 1 < e2e_steps:
            nxt = (i + 1) % 2
            with torch.cuda.stream(copy_stream):
                if i >= 1:
                    copy_stream.wait_event(free[nxt])
                upload(nxt)
                ready[nxt].record(copy_stream)
        compute.wait_event(ready[cur])
        outs = step(bufs[cur])
        free[cur].record(compute)
        d2h_stream.wait_stream(compute)
        with torch.cuda.stream(d2h_stream):
            for h, o in zip(host_out, outs):
                o.record_stream(d2h_stream)   # the allocator keeps o until its D2H is done
                h.copy_(o, non_blocking=True)
    compute.wait_stream(d2h_stream)
    e_end.record(compute)
    barrier(ctx)
    e2e_ms = max_over_ranks(ctx, e_start.elapsed_time(e_end) / e2e_steps)

    if ctx.rank_id != 0:
        return
    pk, pk_src = peaks()
    clocks = clk.summary()
    samples = W["samples_per_step"]
    value = samples / (ms / 1000.0)
    # per-kernel (entry point x layer) records, max launch time over ranks
    merged = {}
    for rk in ranks_k:
        for key, d in rk["ksum"].items():
            m = merged.setdefault(key, {"launches": d["launches"], "ms": 0.0,
                                        "flops": d["flops"], "bytes": d.get("bytes", 0)})
            m["ms"] = max(m["ms"], d["ms"])
    roof = None
    if not merged and W.get("hbm_bytes_per_step"):
        # data-movement workload (cfg5): the pack / unpack / copy kernels are the
        # step; algorithmic HBM bytes (read + write of every element moved) per
        # device-timed step against the measured copy bandwidth
        gbs = W["hbm_bytes_per_step"] / (ms / 1000.0) / 1e9
        hbm = pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
        roof = {"bound": "hbm", "kernel": "copy_rows (redistribute pack / unpack)",
                "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                "traffic": None, "peak_kind": f"{pk_src} HBM copy bandwidth",
                "bytes_per_step": W["hbm_bytes_per_step"]}
    peak, peak_kind = pick_peak(pk, clocks, W["dtype"])
    per_kernel = {}
    for key, d in merged.items():
        avg = d["ms"] / d["launches"]
        ach = (d["flops"] / d["launches"]) / (avg / 1000.0) / 1e12
        per_kernel[key] = {"launches_per_step": d["launches"] / args.steps, "avg_ms": avg,
                           "tflops": ach, "frac": ach / peak,
                           "share_of_step": d["ms"] / args.steps / ms}
        if d.get("bytes"):    # HBM-bound data movement (the bf16x3 operand split)
            gbs = (d["bytes"] / d["launches"]) / (avg / 1000.0) / 1e9
            hbm = pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
            per_kernel[key].update({"gbs": gbs, "frac": gbs / hbm, "bound": "hbm"})
    tensor_keys = {k: v for k, v in merged.items() if not v.get("bytes")}
    if tensor_keys:
        key, d = max(tensor_keys.items(), key=lambda kv: kv[1]["ms"])
        pk_ = per_kernel[key]
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            # per-launch DRAM bytes of this kernel from the committed `ncu --set
            # full` capture (scripts/ncu_summary.py), keyed like `kernels` below
            with open(tpath) as f:
                traffic = json.load(f).get(args.config, {}).get(key)
        roof = {"bound": "tensor", "kernel": key, "achieved": pk_["tflops"], "peak": peak,
                "unit": "TFLOP/s", "frac": pk_["frac"], "traffic": traffic,
                "peak_kind": f"{pk_src} {peak_kind}", "avg_launch_ms": pk_["avg_ms"],
                "flops_per_launch": d["flops"] / d["launches"],
                "timing": "CUDA events around every launch inside the timed steps, "
                          "max over ranks"}
    cpu = None
    if not args.no_cpu_baseline and ctx.mesh.world_size == 1:
        # repeat the one-core sample until ~10 s of CPU work (at most 200 repeats)
        dt = frac = 0.0
        reps = 0
        while reps < 200 and (reps == 0 or dt < 10.0):
            d1, f1 = cpu_fn(1)
            dt += d1
            frac += f1
            reps += 1
        cpu = {"value": frac / dt, "unit": W["unit"], "cores": 1, "kind": "port",
               "sample": f"{reps} x ({sample_desc})", "seconds": dt}
    backend = getattr(ctx.transport, "kind", "thread")
    shared = os.environ.get("DP_MESH_BACKEND") == "gloo-cuda"
    line = {
        "metric": METRIC,
        "value": value, "unit": W["unit"], "n_gpus": ctx.mesh.world_size, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": W["scaling"], "vs_baseline": None, "dtype": W["dtype"],
        "data": "synthetic (torch.randn on device, fixed seeds)", "config": W["info"],
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": samples / (e2e_ms / 1000.0), "unit": W["unit"], "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "note": "pinned H2D of each step's input shards (prefetched one step ahead on "
                        "a copy stream) + D2H of the step's result (drained on a second copy "
                        "stream under the next step), through the public API"},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "simt_calls": sum(rk["simt"] for rk in ranks_k),
        "clocks": clocks,
        "tflops_step": W["flops"] / (ms / 1000.0) / 1e12 if W["flops"] else None,
        "kernels": per_kernel,
        "step_breakdown": {
            "kernel_ms_per_step_by_rank": [rk["kernel_ms"] for rk in ranks_k],
            "ms_per_step_by_rank": [rk["ms"] for rk in ranks_k],
            "non_kernel_ms_per_step_by_rank": [rk["ms"] - rk["kernel_ms"] for rk in ranks_k],
            "note": "non-kernel = step time not covered by conv / attention launches: "
                    "exposed exchange waits, copy / accumulate kernels, weight images"},
        "comm": {"backend": backend + (" (ranks share one GPU: dry run)" if shared else ""),
                 "bytes_sent_per_step_by_rank": [rk["comm_bytes"] for rk in ranks_k]},
    }
    if any(rk["nccl_ms"] for rk in ranks_k):
        # point-to-point rounds timed on the comm stream (CUDA events around
        # each grouped NCCL round): bytes sent / round time per rank, against
        # NVLink 5's 900 GB/s per direction
        nv = []
        for rk in ranks_k:
            gbs = rk["nccl_bytes"] / (rk["nccl_ms"] / 1000.0) / 1e9 if rk["nccl_ms"] else None
            nv.append({"ms_per_step": rk["nccl_ms"], "bytes_per_step": rk["nccl_bytes"],
                       "gbs": gbs, "frac_of_nvlink": gbs / 900.0 if gbs else None})
        line["comm"]["nvlink"] = nv
    if W.get("extra"):
        line["comm"].update(W["extra"])
    print(json.dumps(line), flush=True)


def gather_all(ctx, obj):
    """Every rank's `obj`, in rank order (host metadata, gloo)."""
    if ctx.mesh.world_size == 1:
        return [obj]
    group = ctx.axis_group()
    return ctx.transport.gather_meta(group.members, group.index, obj)


_OPEN = []


def _shutdown():
    for ctx in _OPEN:
        close = getattr(ctx.transport, "close", None)
        if close is not None:
            try:
                close()
            except Exception:  # noqa: BLE001 - best effort at exit
                pass
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
    except Exception:  # noqa: BLE001 - best effort at exit
        pass


if __name__ == "__main__":
    try:
        main()
    finally:
        _shutdown()
