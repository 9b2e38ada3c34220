# cfg1 bf16x3 wgrad ablations (DP_CONV_DBG: 1 no transpose, 2 no MMA, 4 no TMA, 3, 5, 6)
for d in 0 1 2 4 3 5 6 0; do echo "dbg=$d $(DP_CONV_DBG=$d timeout 120 python scripts/x3_wgrad_time.py 2>&1 | tail -1)"; done
