for d in ${DBGS:-0 1 2 4 8 14 15}; do
  DP_CONV_DBG=$d timeout 60 python scripts/conv_time.py fwd 32 32 >> gpurun_out/pair_time.log 2>&1
done
cat gpurun_out/pair_time.log
