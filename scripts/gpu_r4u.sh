# cfg4 SS wgrad: w' tile (K steps) and X ring depth sweep
for kt in 16 12 10 8 6 4; do for nx in 64 6 5 4; do DP_WGRAD_KT=$kt DP_WGRAD_SSNX=$nx timeout 60 python scripts/wgrad_ss_time.py 2>&1 | tail -1; done; done
