# Final verification: the GPU suite, smoke(), the headline bench and the recurrent line.
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
timeout 300 python bench.py --recurrent --no-cpu --steps 10 > gpurun_out/final/bench_c3_recurrent.json 2>&1
for f in bench_c3 bench_c3_recurrent; do python tools/bench_summary.py gpurun_out/final/$f.json 2>/dev/null | head -1; done
