# attention MMAs issued per K-step group (one elect per 4 / 8 MMAs): parity + timings
T=${1:-r4l}
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python scripts/attn_time.py 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_layers.py -q -x -k "attn or ring or cfg3 or vit" 2>&1 | tail -2
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${T}_cfg3.json; python -c "
import json; d=json.load(open('gpurun_out/${T}_cfg3.json')); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k: (round(v['avg_ms'],3), round(v['frac'],3)) for k,v in d['kernels'].items()})"
