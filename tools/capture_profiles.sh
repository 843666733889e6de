#!/bin/bash
# One GPU call's worth of evidence for profiles/: bench lines, reference arm, ncu launch
# list, ncu --set full captures of the main kernels.  Usage (on the GPU box):
#   bash tools/capture_profiles.sh <tag>
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu --steps 10 > $O/bench_c4.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --profile > /dev/null 2>&1
for K in input_proj grad_gemm forward_chunk chunk_scan xbar_chunk; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $O/ncu_$K python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:alif_carry -s 6 -c 2 \
  -o $O/ncu_alif_carry python bench.py --config c4 --steps 1 --warmup 3 --profile > /dev/null 2>&1
ls -la $O
