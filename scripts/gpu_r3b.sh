# ncu launch lists + --set full captures for every config, summarised on the box
# (profiles-ready markdown + traffic.json keyed by the bench names); the .ncu-rep
# files are deleted so gpurun_out/ stays small
T=${1:-r3b}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/${T}_cfg2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/${T}_cfg1_launches.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/${T}_cfg4_launches.csv python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/${T}_cfg3_launches.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in cfg1 cfg2 cfg3 cfg4; do python scripts/ncu_summary.py launches gpurun_out/${T}_${c}_launches.csv gpurun_out/${T}_${c}_launches.md > /dev/null; done
cp profiles/traffic.json gpurun_out/${T}_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_tc_kernel|conv_wgrad_t' -s 12 -c 6 -o /tmp/${T}_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg2.ncu-rep gpurun_out/${T}_cfg2_ncu_full.md --traffic gpurun_out/${T}_traffic.json cfg2 --names "conv_fwd[16->32],conv_fwd[32->32],conv_dgrad[32->32],conv_wgrad[32->32],conv_dgrad[16->32],conv_wgrad[16->32]" > /dev/null
timeout 900 ncu --set full --clock-control none -k regex:'conv_tc_kernel|conv_wgrad_tc_kernel' -s 24 -c 12 -o /tmp/${T}_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg4.ncu-rep gpurun_out/${T}_cfg4_ncu_full.md --traffic gpurun_out/${T}_traffic.json cfg4 --names "conv_fwd[64->64],conv_fwd[64->64],conv_fwd[64->64],conv_fwd[64->64],conv_dgrad[64->64],conv_wgrad[64->64],conv_dgrad[64->64],conv_wgrad[64->64],conv_dgrad[64->64],conv_wgrad[64->64],conv_dgrad[64->64],conv_wgrad[64->64]" > /dev/null
timeout 900 ncu --set full --clock-control none -k regex:'x3_split_act|conv_tc_kernel|conv_wgrad_ts' -s 15 -c 5 -o /tmp/${T}_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg1.ncu-rep gpurun_out/${T}_cfg1_ncu_full.md --traffic gpurun_out/${T}_traffic.json cfg1 --names "x3_split[fp32->3xbf16],conv_fwd[32->32],x3_split[fp32->3xbf16],conv_dgrad[32->32],conv_wgrad[32->32]" > /dev/null
S=65536 timeout 900 ncu --set full --clock-control none -k regex:attn_.*_tc -c 2 -o /tmp/${T}_cfg3 python scripts/attn_prof.py > /dev/null 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg3.ncu-rep gpurun_out/${T}_cfg3_ncu_full.md --traffic gpurun_out/${T}_traffic.json cfg3 --names "attn_fwd_update[d64],attn_bwd_update[d64]" > /dev/null
# the cfg2 conv report's raw metrics, for later reading here
ncu -i /tmp/${T}_cfg2.ncu-rep --page raw --csv > gpurun_out/${T}_cfg2_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | grep ${T}; cat gpurun_out/${T}_traffic.json
