# TS-form (A in TMEM) 32 -> 16 dgrad: parity + A/B against the SS CTA-pair kernel
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc" > gpurun_out/r3k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests.log
tail -5 gpurun_out/r3k_tests.log
for i in 1 2; do for v in 1 0; do echo "tsa=$v"; DP_CONV_TSA=$v timeout 120 python scripts/conv_time.py dgrad 16 32; done; done
timeout 900 python -m pytest tests/test_gpu_tc_sharded.py tests/test_gpu_sharded.py -q -x > gpurun_out/r3k_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests2.log
tail -3 gpurun_out/r3k_tests2.log
for i in 1 2; do for v in 1 0; do DP_CONV_TSA=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tsa=$v', round(d['ms_per_step'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done; done
