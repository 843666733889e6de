#!/bin/bash
# One GPU call's worth of evidence for profiles/: bench lines (C2-C5, reference arm), ncu
# launch lists, ncu --set full captures of every main kernel, the C5 memory sweep and the
# tcgen05 MMA microbenchmark.  Usage (on the GPU box):  bash tools/capture_profiles.sh <tag>
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu --steps 10 > $O/bench_c4.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2.json 2>&1
timeout 300 python bench.py --config c5 --no-cpu --steps 5 > $O/bench_c5.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2>&1
timeout 300 python bench.py --recurrent --no-cpu --steps 5 > $O/bench_c3_recurrent.json 2>&1
timeout 300 python tools/proj_probe.py > $O/proj_probe.txt 2>&1
[ -x tools/mma_pattern_bench ] && ./tools/mma_pattern_bench > $O/mma_pattern_bench.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --profile > /dev/null 2>&1
for K in input_proj grad_gemm forward_chunk chunk_scan xbar_chunk; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $O/ncu_$K python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:alif_carry -s 6 -c 2 \
  -o $O/ncu_alif_carry python bench.py --config c5 --steps 1 --warmup 3 --profile > /dev/null 2>&1
timeout 600 python tools/mem_sweep.py --batch 64 --hidden 256,1024,4096,8192 --T 100,1000,10000 \
  > $O/mem_sweep_c5.jsonl 2>&1
[ -x tools/mma_microbench ] && ./tools/mma_microbench > $O/mma_microbench.txt 2>&1
ls -la $O
