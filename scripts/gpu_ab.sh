# A/B timing of library variants on one box: VARIANTS="head aug" (paper_2605_11111_b200/libdpb200_<v>.so)
cp paper_2605_11111_b200/libdpb200.so /tmp/libdpb200_cur.so
for rep in 1 2; do
for v in ${VARIANTS}; do
  cp paper_2605_11111_b200/libdpb200_$v.so paper_2605_11111_b200/libdpb200.so
  echo "== $v" ; timeout 120 python scripts/attn_time.py; DP_ATTN_TRACE=1 timeout 60 python scripts/attn_prof.py 2>&1 | tail -5; S=65536 timeout 120 python scripts/attn_time.py
done
done
cp /tmp/libdpb200_cur.so paper_2605_11111_b200/libdpb200.so
