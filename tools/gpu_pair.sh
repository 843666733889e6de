# K6p bring-up: pair-vs-single test first (bounded), then the parity suites and the Tc sweep.
mkdir -p gpurun_out/k6p
timeout 300 python -m pytest tests/test_variants_gpu.py -q -x -k carry_pair -p no:cacheprovider > gpurun_out/k6p/pair_test.log 2>&1
echo "pair test rc=$?"; tail -15 gpurun_out/k6p/pair_test.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/k6p/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/k6p/pytest_gpu.log | tail -2; grep -E "^FAILED" gpurun_out/k6p/pytest_gpu.log | head
for pair in 1 0; do
  SPB_CARRY_PAIR=$pair timeout 600 python tools/tc_sweep.py --T 2000 --chunks 127,255,511,1023 > gpurun_out/k6p/tc_sweep_pair$pair.jsonl 2>&1
  echo "pair=$pair"; cat gpurun_out/k6p/tc_sweep_pair$pair.jsonl
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:alif_carry_pair -s 1 -c 1 \
  -o gpurun_out/k6p/ncu_pair_tc511 python tools/tc_sweep.py --T 2000 --chunks 511 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/k6p/ncu_pair_tc511.ncu-rep
