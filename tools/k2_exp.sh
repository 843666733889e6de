python -m pytest tests/test_parity_gpu.py tests/test_headline_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in c3 c4 c5; do python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json | head -3; done
SPB_K2_BANDS=1 python bench.py --no-cpu > gpurun_out/bench_c3_b1.json 2>/dev/null; python tools/bench_summary.py gpurun_out/bench_c3_b1.json | head -2
