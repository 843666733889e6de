# K1 / scan change: the dynamics + parity suites (bounded), then C3 / C5 T=10000 lines.
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_headline_gpu.py tests/test_reset_gpu.py tests/test_variants_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do python bench.py --no-cpu --no-e2e --no-parity > gpurun_out/k1_c3_$r.json 2>/dev/null; python tools/bench_summary.py gpurun_out/k1_c3_$r.json 2>/dev/null | head -5; done
python bench.py --config c5 --seq-len 10000 --no-cpu --no-e2e --no-parity --steps 3 > gpurun_out/k1_c5.json 2>/dev/null; python tools/bench_summary.py gpurun_out/k1_c5.json 2>/dev/null | head -5
