# Launch list of the cfg2 step + ncu --set full of the conv kernels (fwd/dgrad/wgrad).
tag=${1:-r1b}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/${tag}_cfg2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'conv_tc_kernel|conv_wgrad_t' -s 12 -c 6 -o gpurun_out/${tag}_conv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1
ls -la gpurun_out | grep ${tag}
