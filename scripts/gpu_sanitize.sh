# compute-sanitizer memcheck over the kernel parity tests (small shapes)
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20"
for k in "conv_tc_fwd_dgrad" "attention_tc_fwd_bwd" "conv_fp32_bf16x3" "x3_split" "copy_strided or accumulate_strided or element_maps" "conv_single_cta"; do
  echo "== $k"
  timeout 1500 $CS python -m pytest tests/test_gpu_kernels.py -q -x -k "$k" -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds|error" | head -8
done
echo "== sharded tc"
timeout 1500 $CS python -m pytest tests/test_gpu_tc_sharded.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|error" | head -8
