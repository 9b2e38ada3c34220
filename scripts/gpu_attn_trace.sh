# per-block event timeline of CTA 0 of the attention backward (DP_ATTN_TRACE)
for d in ${DBGS:-0}; do
  echo "== dbg=$d" >> gpurun_out/attn_trace.log
  DP_ATTN_DBG=$d DP_ATTN_TRACE=1 timeout 120 python scripts/attn_prof.py >> gpurun_out/attn_trace.log 2>&1
done
cat gpurun_out/attn_trace.log
