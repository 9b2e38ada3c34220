timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/full_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/full_pytest.log
tail -30 gpurun_out/full_pytest.log
