# grouped MMA issue (one elect per 8 K steps) in the three weight-gradient kernels:
# full GPU suite, then cfg1 / cfg2 / cfg4 bench lines
T=${1:-r4k}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -2 gpurun_out/${T}_tests.log
timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -1
for c in cfg2 cfg4 cfg1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${T}_$c.json; python -c "
import json; d=json.load(open('gpurun_out/${T}_$c.json')); print('$c', d['ms_per_step'], d['clocks']['sm_mhz'], {k: (round(v['avg_ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})"; done
for c in "wgrad 16 32" "wgrad 32 32"; do timeout 120 python scripts/conv_time.py $c 2>&1 | tail -1; done
