nproc > gpurun_out/r2e_nproc.txt; free -g >> gpurun_out/r2e_nproc.txt
timeout 900 python -m pytest tests/test_gpu_dispatch.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py -q --durations=10 > gpurun_out/r2e_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_full.log
tail -40 gpurun_out/r2e_full.log; cat gpurun_out/r2e_nproc.txt
