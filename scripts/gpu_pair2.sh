timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv" 2>&1 | tail -2
for w in "fwd 16 32" "fwd 32 32" "dgrad 16 32" "dgrad 32 32"; do
  for e in 0 1; do DP_CONV_2CTA=$e timeout 60 python scripts/conv_time.py $w; done
done
python scripts/conv_time_f32.py
