# cfg3 launch list + ncu --set full of the attention blocks at the bench size (64k x 64k x 16)
tag=${1:-r1g}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv \
    --log-file gpurun_out/${tag}_cfg3_launches.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch3.log 2>&1
S=65536 timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_.*_tc -c 2 \
    -o gpurun_out/${tag}_attn64 python scripts/attn_prof.py > gpurun_out/${tag}_ncu_attn64.log 2>&1
ls -la gpurun_out | grep ${tag}
