#!/bin/bash
# Copy the judged evidence of a capture (tools/capture_profiles.sh) from gpurun_out/<tag>
# to profiles/<tag>: bench lines, launch lists (+ per-kernel shares), ncu summaries and
# SASS hot spots (the .ncu-rep files themselves stay in gpurun_out: too large for git).
set -u
TAG=${1:-r2}
S=gpurun_out/$TAG
D=profiles/$TAG
mkdir -p $D
cp $S/gpu.txt $S/bench_*.json $S/mem_sweep_c5.jsonl $S/c5_sweep.jsonl $S/tc_sweep_*.jsonl $D/ 2>/dev/null
cp $S/mma_microbench.txt $S/mma_pattern_bench.txt $S/proj_probe.txt $S/k2_bands_c3.txt $S/dropin_profile.txt $S/step_timeline_c3.txt $D/ 2>/dev/null
for f in $S/launches_*.csv; do
  b=$(basename $f .csv)
  cp $f $D/
  python tools/launch_summary.py $f > $D/$b.summary.txt
done
for r in $S/ncu_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  { python tools/ncu_summary.py $r; python tools/ncu_hotspots.py $r 20; } > $D/$b.summary.txt 2>&1
done

python tools/traffic_json.py $S > $D/traffic.json
ls -la $D
