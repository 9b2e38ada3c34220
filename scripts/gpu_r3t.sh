# G3 x3 wgrad: pairing order small-first; flush-group size vs precision / time
for r in 1 2 4; do echo "rf_rows=$r"; DP_WGRAD_RF_ROWS=$r timeout 120 python scripts/x3_wgrad_time.py; DP_WGRAD_RF_ROWS=$r timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -1; done
echo "old path:"; DP_WGRAD_G3=0 timeout 120 python scripts/x3_wgrad_time.py; DP_WGRAD_G3=0 timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -1
