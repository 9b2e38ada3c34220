# conv ablations (DP_CONV_DBG: 1 no stores, 2 no MMA, 4 no TMA, 8 no TMEM drain) on the cfg2 layer shapes
for w in "fwd 16 32" "dgrad 16 32" "fwd 32 32"; do
  for d in 0 1 2 4 8 9 12 13 6 14; do DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py $w; done
done > gpurun_out/r2o_abl.txt 2>&1
cat gpurun_out/r2o_abl.txt
