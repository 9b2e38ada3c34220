# TS wgrad: wrapped ring rows issued as two grouped MMA runs
T=${1:-r4n}
mkdir -p gpurun_out
for i in 1 2 3; do timeout 120 python scripts/x3_wgrad_time.py 2>&1 | tail -1; done
timeout 120 python scripts/x3_wgrad_err.py 2>&1 | tail -1
for c in "wgrad 16 32" "wgrad 32 32"; do timeout 120 python scripts/conv_time.py $c 2>&1 | tail -1; done
timeout 1200 python -m pytest tests -m gpu -q -x -k "conv or wgrad or x3 or cfg1 or cfg2 or sharded or fullsize" 2>&1 | tail -2
