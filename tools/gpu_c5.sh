# C5 evidence: K6p pair test, Tc sweep at T = 10000 (K6 per chunk length), ncu of a full
# K6p launch at Tc = 511 and 2047, then the C5 grid (hidden x T at B = 256).
mkdir -p gpurun_out/c5
timeout 300 python -m pytest tests/test_variants_gpu.py -q -x -k carry_pairs -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/tc_sweep.py --T 10000 --chunks 511,1023,2047 > gpurun_out/c5/tc_sweep_T10000.jsonl 2>&1
timeout 600 python tools/tc_sweep.py --T 2000 --chunks 255,511,1023 > gpurun_out/c5/tc_sweep_T2000.jsonl 2>&1
cat gpurun_out/c5/tc_sweep_*.jsonl
for TC in 511 2047; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:alif_carry -s 1 -c 1 \
    -o gpurun_out/c5/ncu_pair_tc$TC python tools/tc_sweep.py --T 10000 --chunks $TC --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/c5/ncu_pair_tc$TC.ncu-rep | head -22
done
timeout 2400 python tools/c5_sweep.py --out gpurun_out/c5/sweep.jsonl > gpurun_out/c5/sweep.log 2>&1
echo "sweep rc=$?"; cat gpurun_out/c5/sweep.jsonl | cut -c1-400
