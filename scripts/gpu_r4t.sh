# HEAD re-check after the bf16x3 wgrad A-ring change: full GPU suite, smoke, cfg1 + cfg2 bench
# lines, cfg1 launch list and ncu --set full summary, traffic.json (cfg1 keys refreshed)
T=${1:-r4t}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python scripts/smoke_launches.py > gpurun_out/${T}_smoke_launches.txt 2>&1
timeout 600 python bench.py > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg1.json 2> gpurun_out/${T}_cfg1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/${T}_cfg1_launches.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_cfg1_launches.csv gpurun_out/${T}_cfg1_launches.md > /dev/null
cp profiles/traffic.json gpurun_out/${T}_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'x3_split_act|conv_tc_kernel|conv_wgrad_ts' -s 15 -c 5 -o /tmp/${T}_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg1.ncu-rep gpurun_out/${T}_cfg1_ncu_full.md --traffic gpurun_out/${T}_traffic.json cfg1 --names "x3_split[fp32->3xbf16],conv_fwd[32->32],x3_split[fp32->3xbf16],conv_dgrad[32->32],conv_wgrad[32->32]" > /dev/null
tail -2 gpurun_out/${T}_tests.log
for c in cfg2 cfg1; do python -c "
import json; d=json.loads(open('gpurun_out/${T}_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['simt_calls'], {k: (round(v['avg_ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})"; done
cat gpurun_out/${T}_cfg1_launches.md | head -12
