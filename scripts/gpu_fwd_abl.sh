for w in "fwd 32 32" "dgrad 32 16" "fwd 16 32"; do
  for d in 0 1 2 4 8 9 6 5 3; do
    DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py $w >> gpurun_out/fwd_abl.log 2>&1
  done
done
cat gpurun_out/fwd_abl.log
