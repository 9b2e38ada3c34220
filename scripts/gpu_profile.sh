# Profile the cfg2 step on one B200: launch list + ncu --set full of the
# three tcgen05 conv kernels.  Outputs land in gpurun_out/<tag>_*.
tag=${1:-prof}
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'conv_tc_kernel|conv_wgrad_tc_kernel' -s 12 -c 6 -o gpurun_out/${tag}_conv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1
ls -la gpurun_out | grep ${tag}
