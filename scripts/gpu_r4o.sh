# A/B (same box, interleaved): TS wgrad wrapped rows grouped (default) vs per-MMA (DP_CONV_DBG=64)
for i in 1 2 3; do for d in 0 64; do for c in "wgrad 16 32" "wgrad 32 32"; do echo "dbg=$d $(DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py $c 2>&1 | tail -1)"; done; done; done
