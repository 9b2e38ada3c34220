# e2e with the D2H drain overlapped (cfg3, cfg2), MUFU ex2 probe
T=${1:-r4d}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_probe scripts/mufu_probe.cu && /tmp/mufu_probe > gpurun_out/${T}_mufu.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/${T}_mufu.log
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg3.json 2> gpurun_out/${T}_cfg3.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
cat gpurun_out/${T}_mufu.log
for c in cfg3 cfg2; do python -c "
import json; d=json.loads(open('gpurun_out/${T}_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])"; done
