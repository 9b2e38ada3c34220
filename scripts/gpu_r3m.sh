# TS-form dgrad: parity + ablations (128 = no TMEM stores, 2 = no MMA) + SS reference
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc" > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log
tail -2 gpurun_out/r3m_tests.log
for d in 0 128 2 0; do echo "dbg=$d"; DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py dgrad 16 32; done
DP_CONV_TSA=0 timeout 120 python scripts/conv_time.py dgrad 16 32
