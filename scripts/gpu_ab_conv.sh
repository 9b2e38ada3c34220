# A/B timing of conv library variants on one box: VARIANTS="a b" (paper_2605_11111_b200/libdpb200_<v>.so)
cp paper_2605_11111_b200/libdpb200.so /tmp/libdpb200_keep.so
for rep in 1 2; do
for v in ${VARIANTS}; do
  cp paper_2605_11111_b200/libdpb200_$v.so paper_2605_11111_b200/libdpb200.so
  echo "== $v"; for w in "fwd 32 32" "fwd 16 32" "dgrad 32 32" "dgrad 16 32"; do python scripts/conv_time.py $w; done
done
done
cp /tmp/libdpb200_keep.so paper_2605_11111_b200/libdpb200.so
