# cfg1 dW row-flush precision fix + conv kernel tests + cfg2 launch list / ncu full capture
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py tests/test_gpu_kernels.py -q -x -k "cfg1 or conv" > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
timeout 300 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_cfg1.json 2> gpurun_out/r2g_cfg1.err
bash scripts/gpu_profile_conv.sh r2g
tail -5 gpurun_out/r2g_tests.log; cat gpurun_out/r2g_cfg1.json; tail -3 gpurun_out/r2g_cfg1.err
