# conv ablations (DP_CONV_DBG: 1 no stores, 2 no MMA, 4 no TMA) for the cfg2 layer shapes
for w in "fwd 16 32" "dgrad 16 32" "fwd 32 32"; do
  for d in 0 1 2 4 5 3 6; do DP_CONV_DBG=$d python scripts/conv_time.py $w; done
done
