# Quick GPU check: selected test files (-x) then bench lines for the given configs.
#   bash tools/gpu_quick.sh "<pytest args>" [configs...]
mkdir -p gpurun_out
T="$1"; shift
python -m pytest $T -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_quick.log | grep -vE "^\s*$" | tail -22
for c in "$@"; do
  python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?"; tail -3 gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json
done
