set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 600 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 6 -c 3 -o gpurun_out/r1_conv_tc python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r1_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad_tc_kernel -s 2 -c 2 -o gpurun_out/r1_wgrad_tc python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r1_ncu_full2.log 2>&1
ls -la gpurun_out
