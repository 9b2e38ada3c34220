for w in "fwd 32 32" "dgrad 16 32"; do
  for d in ${DBGS:-0 5 21 16}; do
    DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py $w >> gpurun_out/fwd_abl.log 2>&1
  done
done
cat gpurun_out/fwd_abl.log
