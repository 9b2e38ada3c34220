# TS wgrad junk-lane zeroing under the power cap: sustained (300-step) A/B, alternating
for i in 1 2; do
  for d in 0 64; do DP_CONV_DBG=$d timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg=$d', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
done
