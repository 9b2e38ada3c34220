# TS-form dgrad, tcgen05.cp variant (DP_CONV_TSA=2): parity + A/B vs stagers (1) and SS (0)
DP_CONV_TSA=2 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc" > gpurun_out/r3n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_tests.log
tail -25 gpurun_out/r3n_tests.log | grep -v "^  " | tail -8
for i in 1 2; do for v in 2 1 0; do echo "tsa=$v"; DP_CONV_TSA=$v timeout 120 python scripts/conv_time.py dgrad 16 32; done; done
