# grouped bf16x3 wgrad (G3): fp32 parity (kernel cases, sharded fp32, cfg1 full grid vs oracle) + A/B
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "fp32 or bf16x3 or x3" > gpurun_out/r3s_t1.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_t1.log; tail -2 gpurun_out/r3s_t1.log
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fullsize_oracle.py -q -x -k "fp32 or cfg1" > gpurun_out/r3s_t2.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_t2.log; tail -2 gpurun_out/r3s_t2.log
for i in 1 2; do for v in 1 0; do echo "g3=$v"; DP_WGRAD_G3=$v timeout 120 python scripts/x3_wgrad_time.py; done; done
for v in 1 0; do DP_WGRAD_G3=$v timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -2; done
for v in 1 0; do DP_WGRAD_G3=$v timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg1 g3=$v', round(d['ms_per_step'],4), {k: (round(v['avg_ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})"; done
