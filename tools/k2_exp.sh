timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "pair_gemm or banded or as_benched or shd" 2>&1 | tail -2
for r in 1 2; do
for v in "" "SPB_K5_BN=256" "SPB_LIB=ab/lib_scan12o7.so" "SPB_LIB=ab/lib_scan16o6.so" "SPB_LIB=ab/lib_scan16o7.so" "SPB_LIB=ab/lib_scan8o8.so"; do
  env $v timeout 300 python bench.py --no-cpu --steps 30 > gpurun_out/ab.json 2>/dev/null
  echo -n "[$v] "; python tools/bench_summary.py gpurun_out/ab.json 2>/dev/null | grep -E "ms=|gemm|forward " | sed -E 's/.*ms=([0-9.]+).*/ms=\1/; s/.hbm_gbs.*//' | tr '\n' ' '; echo
done; done
