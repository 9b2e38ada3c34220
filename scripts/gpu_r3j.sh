# bulk-store conv epilogue: parity + A/B (cfg2, cfg4, standalone shapes)
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tc_sharded.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py -q -x > gpurun_out/r3j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3j_tests.log
tail -3 gpurun_out/r3j_tests.log
for w in "fwd 16 32" "fwd 32 32" "dgrad 32 32" "dgrad 16 32"; do for v in 1 0; do DP_CONV_BSTORE=$v timeout 120 python scripts/conv_time.py $w; done; done
for i in 1 2; do for v in 1 0; do DP_CONV_BSTORE=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bstore=$v', round(d['ms_per_step'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done; done
for v in 1 0; do DP_CONV_BSTORE=$v timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 bstore=$v', round(d['ms_per_step'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
