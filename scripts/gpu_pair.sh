timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv_tc" > gpurun_out/pair_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pair_pytest.log
tail -25 gpurun_out/pair_pytest.log
for w in "fwd 16 32" "fwd 32 32" "dgrad 16 32" "dgrad 32 32"; do
  for e in 0 1; do
    DP_CONV_PAIR=$e timeout 60 python scripts/conv_time.py $w >> gpurun_out/pair_time.log 2>&1
  done
done
cat gpurun_out/pair_time.log
