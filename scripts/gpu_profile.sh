# Profile one B200: launch lists for cfg2 / cfg3 steps and ncu --set full of
# the tcgen05 conv + attention kernels.  Outputs land in gpurun_out/<tag>_*.
tag=${1:-prof}
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/${tag}_cfg2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv \
    --log-file gpurun_out/${tag}_cfg3_launches.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'conv_tc_kernel|conv_wgrad_tc_kernel' -s 12 -c 6 -o gpurun_out/${tag}_conv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -c 2 \
    -o gpurun_out/${tag}_attn python scripts/attn_prof.py > gpurun_out/${tag}_ncu_attn.log 2>&1
ls -la gpurun_out | grep ${tag}
