timeout 900 python -m pytest tests/test_gpu_layers.py -x -q > gpurun_out/layers_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/layers_pytest.log
tail -30 gpurun_out/layers_pytest.log
