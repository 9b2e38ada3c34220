# x3 wgrad ablation: RF drain work skipped (DP_CONV_DBG=64) alone and with no transposes (65)
for d in 0 64 1 65 5 69 0; do echo "dbg=$d $(DP_CONV_DBG=$d timeout 120 python scripts/x3_wgrad_time.py 2>&1 | tail -1)"; done
