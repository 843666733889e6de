# K6 evidence: the Tc sweep at C5 shape (T = 2000 and 10000) and ncu captures of full
# carry launches at Tc = 511 and 2047.
mkdir -p gpurun_out/k6
python tools/tc_sweep.py --T 2000 > gpurun_out/k6/tc_sweep_T2000.jsonl 2>&1
python tools/tc_sweep.py --T 10000 --chunks 511,1023,2047 > gpurun_out/k6/tc_sweep_T10000.jsonl 2>&1
cat gpurun_out/k6/*.jsonl
for TC in 511 2047; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:alif_carry -s 1 -c 1 \
    -o gpurun_out/k6/ncu_carry_tc$TC python tools/tc_sweep.py --T 10000 --chunks $TC --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/k6/ncu_carry_tc$TC.ncu-rep
done
python tools/dropin_profile.py > gpurun_out/k6/dropin_profile.txt 2>&1; head -40 gpurun_out/k6/dropin_profile.txt
