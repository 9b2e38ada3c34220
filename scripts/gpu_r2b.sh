timeout 900 python -m pytest tests/test_gpu_tc_sharded.py -x -q > gpurun_out/r2b_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tc.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_gpu.log
timeout 300 python scripts/smoke_launches.py > gpurun_out/r2b_smoke_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_smoke_launches.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
tail -5 gpurun_out/r2b_tc.log; tail -5 gpurun_out/r2b_gpu.log; cat gpurun_out/r2b_smoke_launches.log | tail -40
