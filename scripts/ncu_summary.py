"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py launches <launches.csv> <out.md>
    python scripts/ncu_summary.py full <report.ncu-rep> <out.md> [--traffic profiles/traffic.json KEY]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list into
per-kernel count / total / share; `full` pulls the counters DESIGN.md cites
(duration, DRAM bytes, tensor-pipe activity, SM clock, registers, smem) from
a `--set full` report, one row per captured launch.
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict


def short(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("dp::", "")
    return name.split("(")[0][:80]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    total = 0.0
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] in ("nsecond", "ns"):
            v /= 1e3
        elif r[ui] in ("msecond", "ms"):
            v *= 1e3
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
    with open(out, "w") as f:
        f.write(f"# Launch list summary ({path})\n\n")
        f.write("ncu `--metrics gpu__time_duration.sum --clock-control none`: cold-cache, serialised "
                "launches; compare SHARES, not absolute times.\n\n")
        f.write("| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {t:.1f} | {t / n:.1f} | {t / total:.1%} |\n")
    print(open(out).read())


FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe % active (realtime)"),
    ("TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
     "hmma subpipe active cycles (avg/SM)"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed (avg)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "smem->tensor wavefronts % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]


def full(path, out, traffic=None, key=None, names=None):
    """names: the bench's kernel keys (e.g. conv_fwd[16->32]) of the captured
    launches in capture order; traffic.json is then keyed by those, which is
    what bench.py looks up for roofline.traffic."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {n: i for i, n in enumerate(hdr)}
    lines = []
    tr = {}
    for r in rows[2:]:
        name = short(r[idx["Kernel Name"]])
        vals = {}
        for m, label in FULL_METRICS:
            if m in idx and r[idx[m]] != "":
                vals[label] = f"{r[idx[m]]} {units[idx[m]]}".strip()
        lines.append((name, vals))
        # per-launch DRAM traffic in bytes
        def to_bytes(m):
            if m not in idx or r[idx[m]] == "":
                return 0.0
            v = float(r[idx[m]].replace(",", ""))
            u = units[idx[m]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        label = names[len(lines) - 1] if names and len(lines) <= len(names) else name
        tr.setdefault(label, []).append(to_bytes("dram__bytes_read.sum") +
                                        to_bytes("dram__bytes_write.sum"))
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({path})\n\n")
        for name, vals in lines:
            f.write(f"## `{name}`\n\n| metric | value |\n|---|---|\n")
            for k, v in vals.items():
                f.write(f"| {k} | {v} |\n")
            f.write("\n")
    print(open(out).read())
    if traffic and key:
        try:
            data = json.load(open(traffic))
        except OSError:
            data = {}
        data[key] = {}
        for name, vals in tr.items():
            data.setdefault(key, {})[name] = sum(vals) / len(vals)
        json.dump(data, open(traffic, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        t = k = None
        if "--traffic" in sys.argv:
            i = sys.argv.index("--traffic")
            t, k = sys.argv[i + 1], sys.argv[i + 2]
        nm = None
        if "--names" in sys.argv:
            nm = sys.argv[sys.argv.index("--names") + 1].split(",")
        full(sys.argv[2], sys.argv[3], t, k, nm)
