for c in "16 32" "32 32"; do
  for d in ${DBGS:-7 71 0 64}; do
    DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py wgrad $c >> gpurun_out/wg_time.log 2>&1
  done
done
cat gpurun_out/wg_time.log
