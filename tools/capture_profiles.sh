#!/bin/bash
# One GPU call's worth of evidence for profiles/: bench lines (C2-C5, the strong-scaling
# C4 point, the reference arm, the recurrent extension), ncu launch lists, ncu --set full
# captures of every main kernel (K6p at the C5 shape, Tc = 511 and 2047), the Tc sweep and
# the C5 grid.  Usage (on the GPU box):  bash tools/capture_profiles.sh <tag>
set -u
TAG=${1:-r2}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu --steps 10 > $O/bench_c4.json 2>&1
timeout 600 python bench.py --config c4 --global-batch 1024 --no-cpu --steps 5 > $O/bench_c4_gb1024.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2.json 2>&1
timeout 300 python bench.py --config c5 --no-cpu --steps 5 > $O/bench_c5.json 2>&1
timeout 600 python bench.py --config c5 --seq-len 10000 --no-cpu --steps 3 > $O/bench_c5_T10000.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2>&1
timeout 300 python bench.py --recurrent --no-cpu --steps 5 > $O/bench_c3_recurrent.json 2>&1
timeout 300 python tools/proj_probe.py > $O/proj_probe.txt 2>&1
timeout 300 python tools/k2_bands.py 1,2,3,4,6,8 8 > $O/k2_bands_c3.txt 2>&1
timeout 300 python tools/dropin_profile.py > $O/dropin_profile.txt 2>&1
timeout 300 python tools/step_timeline.py --out $O/step_timeline_c3.json > $O/step_timeline_c3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c5_T10000.csv python bench.py --config c5 --seq-len 10000 --steps 1 --warmup 3 --profile > /dev/null 2>&1
for K in input_proj grad_gemm forward_chunk chunk_scan; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $O/ncu_$K python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1
done
for TC in 511 2047; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:alif_carry -s 1 -c 1 \
    -o $O/ncu_alif_carry_tc$TC python tools/tc_sweep.py --T 10000 --chunks $TC --reps 1 > /dev/null 2>&1
done
timeout 900 python tools/tc_sweep.py --T 10000 --chunks 255,511,1023,2047 > $O/tc_sweep_T10000.jsonl 2>&1
timeout 600 python tools/tc_sweep.py --T 2000 --chunks 127,255,511,1023,2047 > $O/tc_sweep_T2000.jsonl 2>&1
timeout 2400 python tools/c5_sweep.py --out $O/c5_sweep.jsonl > $O/c5_sweep.log 2>&1
ls -la $O
