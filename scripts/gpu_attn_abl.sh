for d in ${DBGS:-0 1 2 4 8 6 10 12 14}; do
  DP_ATTN_DBG=$d timeout 120 python scripts/attn_time.py >> gpurun_out/attn_abl.log 2>&1
done
cat gpurun_out/attn_abl.log
