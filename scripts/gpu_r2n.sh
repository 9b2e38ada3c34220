# evidence: smoke launch list (no at:: / SIMT kernels), self-launched multi-rank bench on the one GPU
# (gloo-cuda; per-rank kernel rates vs N=1), cfg5 size sweep at N=1
timeout 600 python scripts/smoke_launches.py > gpurun_out/r2n_smoke_launches.txt 2>&1
for n in 2 4; do
  timeout 900 python bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_cfg2_g$n.json 2> gpurun_out/r2n_cfg2_g$n.err
done
timeout 900 python bench.py --gpus 2 --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_cfg3_g2.json 2> gpurun_out/r2n_cfg3_g2.err
timeout 900 python bench.py --gpus 2 --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_cfg4_g2.json 2> gpurun_out/r2n_cfg4_g2.err
for s in 64 256 1024 4096 8192; do
  timeout 600 python bench.py --config cfg5 --size-mib $s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_cfg5_$s.json 2> gpurun_out/r2n_cfg5_$s.err
done
head -40 gpurun_out/r2n_smoke_launches.txt
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r2n_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("n_gpus"), d.get("ms_per_step"), d.get("value"), {k: (round(v["avg_ms"], 4), round(v.get("frac", 0), 3)) for k, v in d.get("kernels", {}).items()}, d.get("roofline", {}).get("frac"))
    except Exception as e:
        print(f, "ERR", e)
PY
