#!/bin/bash
# The parts of tools/capture_profiles.sh a K2/step change touches (the C5 grid and the Tc
# sweeps are not re-run), plus the GPU suite and smoke():  bash tools/capture_refresh.sh r2
set -u
TAG=${1:-r2}
O=gpurun_out/$TAG
mkdir -p $O
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu --steps 10 > $O/bench_c4.json 2>&1
timeout 600 python bench.py --config c4 --global-batch 1024 --no-cpu --steps 5 > $O/bench_c4_gb1024.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2.json 2>&1
timeout 300 python bench.py --config c5 --no-cpu --steps 5 > $O/bench_c5.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2>&1
timeout 300 python bench.py --recurrent --no-cpu --steps 5 > $O/bench_c3_recurrent.json 2>&1
timeout 300 python tools/proj_probe.py > $O/proj_probe.txt 2>&1
timeout 300 python tools/k2_bands.py 1,2,3,4,6,8 8 > $O/k2_bands_c3.txt 2>&1
timeout 300 python tools/dropin_profile.py > $O/dropin_profile.txt 2>&1
timeout 300 python tools/step_timeline.py --out $O/step_timeline_c3.json 2>&1 | grep -v -i warn > $O/step_timeline_c3.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --profile > /dev/null 2>&1
for K in input_proj readout_loss; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $O/ncu_$K -f python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1
done
for f in bench_c3 bench_c4 bench_c4_gb1024 bench_c2 bench_c5 bench_c3_recurrent; do
  python tools/bench_summary.py $O/$f.json 2>/dev/null | head -1
done
ls -la $O | wc -l
