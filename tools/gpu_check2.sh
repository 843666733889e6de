# GPU suite + bench lines (C3, C3 recurrent, C5 at T = 10000) + the K6 Tc sweep.
mkdir -p gpurun_out/chk
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/chk/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/chk/pytest_gpu.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/chk/pytest_gpu.log | head
python bench.py --no-cpu > gpurun_out/chk/bench_c3.json 2>/dev/null; python tools/bench_summary.py gpurun_out/chk/bench_c3.json | head -2
python bench.py --recurrent --no-cpu --no-e2e --steps 10 > gpurun_out/chk/bench_rec.json 2>/dev/null; python tools/bench_summary.py gpurun_out/chk/bench_rec.json | head -3
python bench.py --config c5 --seq-len 10000 --no-cpu --no-e2e --steps 3 > gpurun_out/chk/bench_c5_T10000.json 2>/dev/null; python tools/bench_summary.py gpurun_out/chk/bench_c5_T10000.json | head -8
