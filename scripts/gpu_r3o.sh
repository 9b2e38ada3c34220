# TS-form dgrad as a CTA pair (cta_group::2, A from each CTA's TMEM): parity + A/B
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc" > gpurun_out/r3o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3o_tests.log
tail -25 gpurun_out/r3o_tests.log | grep -v "^  " | tail -6
for i in 1 2; do for v in 1 0; do echo "tsa=$v"; DP_CONV_TSA=$v timeout 120 python scripts/conv_time.py dgrad 16 32; done; done
for d in 128 2; do echo "dbg=$d"; DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py dgrad 16 32; done
