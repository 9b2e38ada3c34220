# cfg3 launch list + ncu --set full of the attention blocks (16k ring-step size), cfg1 launch list
tag=${1:-r1c}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv \
    --log-file gpurun_out/${tag}_cfg3_launches.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv \
    --log-file gpurun_out/${tag}_cfg1_launches.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -c 2 \
    -o gpurun_out/${tag}_attn python scripts/attn_prof.py > gpurun_out/${tag}_ncu_attn.log 2>&1
ls -la gpurun_out | grep ${tag}
