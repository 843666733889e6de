# compute-sanitizer memcheck over small GPU tests of the pair kernels and the engine paths
mkdir -p gpurun_out/san
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_variants_gpu.py -q -x -p no:cacheprovider -k "carry_pairs and (256-130 or 384-700 or lif)" > gpurun_out/san/memcheck_k6.log 2>&1
echo "memcheck k6 rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/san/memcheck_k6.log | head -5
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "pair_gemm or batched_vs_two_pass" > gpurun_out/san/memcheck_k5.log 2>&1
echo "memcheck k5 rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/san/memcheck_k5.log | head -5
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_recurrent_gpu.py tests/test_reset_gpu.py -q -x -p no:cacheprovider > gpurun_out/san/memcheck_rec.log 2>&1
echo "memcheck rec/reset rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/san/memcheck_rec.log | head -5
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "projection or int8 or binary or pooled" > gpurun_out/san/memcheck_k2.log 2>&1
echo "memcheck k2 rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/san/memcheck_k2.log | head -5
