# attention backward: dQ drained to registers before the staging wait (TMEM freed at once)
T=${1:-r4f}
mkdir -p gpurun_out
timeout 300 python scripts/attn_time.py > gpurun_out/${T}_quick.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_quick.log
tail -2 gpurun_out/${T}_quick.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py -q -x -k "attn or ring or cfg3" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -2 gpurun_out/${T}_tests.log
for i in 1 2 3; do timeout 300 python scripts/attn_time.py 2>&1 | tail -1; done
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg3.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/${T}_cfg3.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})"
