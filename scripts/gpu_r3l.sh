# TS-form dgrad iteration: parity + standalone A/B
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc" > gpurun_out/r3l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3l_tests.log
tail -2 gpurun_out/r3l_tests.log
for i in 1 2; do for v in 1 0; do echo "tsa=$v"; DP_CONV_TSA=$v timeout 120 python scripts/conv_time.py dgrad 16 32; done; done
