timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2c_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_gpu.log
timeout 300 python scripts/smoke_launches.py > gpurun_out/r2c_smoke_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_smoke_launches.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench2.json 2> gpurun_out/r2c_bench2.err
tail -15 gpurun_out/r2c_gpu.log; cat gpurun_out/r2c_smoke_launches.log | tail -30; cat gpurun_out/r2c_bench.json; tail -3 gpurun_out/r2c_bench.err; cat gpurun_out/r2c_bench2.json; tail -5 gpurun_out/r2c_bench2.err
