# One gpurun call: the GPU test suite, bench lines for the given configs, the reference arm.
#   bash tools/gpu_check.sh [configs...]     (default: c3)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -3
grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu.log | head -20
for c in ${@:-c3}; do
  python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?"; python tools/bench_summary.py gpurun_out/bench_$c.json
done
