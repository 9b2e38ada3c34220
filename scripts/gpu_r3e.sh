# TS wgrad without mirrored X slots (wrap rows as two MMAs): parity + timing
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tc_sharded.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py -q -x > gpurun_out/r3e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_tests.log
tail -3 gpurun_out/r3e_tests.log
for i in 1 2; do timeout 120 python scripts/conv_time.py wgrad 16 32; timeout 120 python scripts/conv_time.py wgrad 32 32; done
timeout 120 python scripts/x3_wgrad_time.py; timeout 120 python scripts/x3_wgrad_err.py
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
