# G3 x3 wgrad final: fp32 parity suites + cfg1 bench A/B
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_fullsize.py tests/test_gpu_tc_sharded.py -q -x > gpurun_out/r3u_t.log 2>&1; echo "rc=$?" >> gpurun_out/r3u_t.log; tail -2 gpurun_out/r3u_t.log
timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -1
for i in 1 2; do for v in 1 0; do DP_WGRAD_G3=$v timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg1 g3=$v', round(d['ms_per_step'],4), {k: (round(v['avg_ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})"; done; done
