# round 2: first GPU pass of this session — full gpu suite, smoke launch list, N=1 bench, N=2 bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2f_gpu.txt; nproc >> gpurun_out/r2f_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2f_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_gpu.log
timeout 300 python scripts/smoke_launches.py > gpurun_out/r2f_smoke_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_smoke_launches.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench2.json 2> gpurun_out/r2f_bench2.err
tail -25 gpurun_out/r2f_gpu.log; tail -30 gpurun_out/r2f_smoke_launches.log; cat gpurun_out/r2f_bench.json; tail -3 gpurun_out/r2f_bench.err; cat gpurun_out/r2f_bench2.json; tail -5 gpurun_out/r2f_bench2.err
