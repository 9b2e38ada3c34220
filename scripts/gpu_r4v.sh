# bf16x3 wgrad: pairings grouped by dY part (shared TMEM A slices), one elect per part
T=${1:-r4s}
mkdir -p gpurun_out
for i in 1 2 3; do timeout 120 python scripts/x3_wgrad_time.py 2>&1 | tail -1; done
timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -1
for d in 1 2 5; do echo "dbg=$d $(DP_CONV_DBG=$d timeout 120 python scripts/x3_wgrad_time.py 2>&1 | tail -1)"; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_sharded.py -q -x -k "x3 or fp32 or cfg1" 2>&1 | tail -2
timeout 300 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${T}_cfg1.json; python -c "
import json; d=json.load(open('gpurun_out/${T}_cfg1.json')); print(d['ms_per_step'], {k: (round(v['avg_ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})"
