# TS wgrad ring depths (dY ring nd, TMEM A slots na) on the cfg2 shapes
for nd in 4 6 8; do for na in 4 6; do
  DP_WGRAD_ND=$nd DP_WGRAD_NA=$na timeout 120 python scripts/conv_time.py wgrad 16 32
  DP_WGRAD_ND=$nd DP_WGRAD_NA=$na timeout 120 python scripts/conv_time.py wgrad 32 32
done; done > gpurun_out/r2t_wgrad_rings.txt 2>&1
cat gpurun_out/r2t_wgrad_rings.txt
