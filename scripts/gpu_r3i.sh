# cfg4 fwd/dgrad on CTA pairs (N = 64): parity + A/B
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tc_sharded.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r3i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3i_tests.log
tail -3 gpurun_out/r3i_tests.log
for i in 1 2; do for v in 1 0; do DP_CONV_PAIR64=$v timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pair64=$v', round(d['ms_per_step'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done; done
