# K5 pair bring-up: GEMM tests (bounded), the full GPU suite, C3/C4/C5 with and without.
mkdir -p gpurun_out/k5p
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "gemm" -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/k5p/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/k5p/pytest_gpu.log | tail -1; grep -E "^FAILED|^ERROR" gpurun_out/k5p/pytest_gpu.log | head
for c in c3 c4 c5; do
  for p in 1 0; do
    SPB_GEMM_PAIR=$p python bench.py --config $c --no-cpu --no-e2e --no-parity --steps 20 > gpurun_out/k5p/b_${c}_$p.json 2>/dev/null
    python - $c $p gpurun_out/k5p/b_${c}_$p.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1]); k=d["kernels"]["gemm"]
print(sys.argv[1], "pair" if sys.argv[2]=="1" else "single", "ms/update", round(d["ms_per_step"],4), "K5 ms", round(k["ms_per_step"],4), "tensor frac", round(k["tensor_frac"],3))
PY
  done
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grad_gemm_pair -s 3 -c 1 \
  -o gpurun_out/k5p/ncu_k5p python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/k5p/ncu_k5p.ncu-rep | head -14
