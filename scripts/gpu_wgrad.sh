# wgrad TS ablations (DP_CONV_DBG bits: 1 no transpose, 2 no MMA, 4 no TMA)
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv_tc" > gpurun_out/wg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/wg_pytest.log
for c in "16 32" "32 32"; do
  for d in ${DBGS:-0 5 6}; do
    DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py wgrad $c >> gpurun_out/wg_time.log 2>&1
  done
done
cat gpurun_out/wg_time.log; tail -2 gpurun_out/wg_pytest.log
