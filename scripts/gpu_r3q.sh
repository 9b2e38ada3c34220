# TS wgrad ablations (DP_CONV_DBG: 1 no transpose, 2 no MMA, 4 no TMA) for the cfg2 shapes
for sh in "16 32" "32 32"; do for d in 0 1 2 4 3 5 6; do echo "wgrad $sh dbg=$d"; DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py wgrad $sh; done; done
