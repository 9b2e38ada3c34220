# attention backward Q/dO multicast over key-tile pairs: parity, then A/B timings
T=${1:-r4e}
mkdir -p gpurun_out
timeout 300 python scripts/attn_time.py > gpurun_out/${T}_quick.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_quick.log
tail -3 gpurun_out/${T}_quick.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py -q -x -k "attn or ring or cfg3" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for i in 1 2; do for mc in 1 0; do echo "MC=$mc $(DP_ATTN_MC=$mc timeout 300 python scripts/attn_time.py 2>&1 | tail -2 | tr '\n' ' ')"; done; done > gpurun_out/${T}_time.log
cat gpurun_out/${T}_time.log
for mc in 1 0; do DP_ATTN_MC=$mc timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg3_mc$mc.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/${T}_cfg3_mc$mc.json').read().strip().splitlines()[-1]); print('MC=$mc', d['ms_per_step'], d['clocks']['sm_mhz'], {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})"; done
