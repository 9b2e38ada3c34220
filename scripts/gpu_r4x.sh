# conv fwd/dgrad (C_in 32 shapes): both 16-channel steps x 3 kw taps under one elect (default) vs
# the 3-MMA groups (DP_CONV_DBG=64), interleaved on one box; parity first
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc or issue_paths or dense_conv" 2>&1 | tail -2
for i in 1 2; do for d in 0 64; do for c in "dgrad 16 32" "fwd 32 32" "dgrad 32 32"; do echo "dbg=$d $(DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py $c 2>&1 | tail -1)"; done; done; done
for i in 1 2; do for d in 0 64; do echo "cfg2 dbg=$d $(DP_CONV_DBG=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})")"; done; done
