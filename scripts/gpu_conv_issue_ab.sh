# grouped (3 kw taps per elect) vs single-MMA issue in the merged conv steps (DP_CONV_DBG=32 = old path)
for rep in 1 2; do
for d in 0 32; do
  DP_CONV_DBG=$d python scripts/conv_time.py fwd 32 32
  DP_CONV_DBG=$d python scripts/conv_time.py fwd 16 32
  DP_CONV_DBG=$d python scripts/conv_time.py dgrad 32 32
  DP_CONV_DBG=$d python scripts/conv_time.py dgrad 16 32
done
done
for d in 0 32; do
  DP_CONV_DBG=$d python bench.py --config cfg4 --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 dbg=$d', round(d['ms_per_step'],3), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
  DP_CONV_DBG=$d python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2 dbg=$d', round(d['ms_per_step'],3), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
done
