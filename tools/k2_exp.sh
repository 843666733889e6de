for r in 1 2 3; do for L in oldloop new; do echo -n "$L: "; SPB_LIB=ab/lib_$L.so python tools/k2_bands.py 4 12 2>&1 | grep bands; done; done
for L in oldloop new; do SPB_LIB=ab/lib_$L.so python bench.py --no-cpu > gpurun_out/bench_$L.json 2>/dev/null; echo $L; python tools/bench_summary.py gpurun_out/bench_$L.json 2>/dev/null| head -2; done
