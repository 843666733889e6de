# A/B of where K5's raw-spike operand is written at C3: folded into the pack (default) vs a
# side-stream K4 overlapping K2 ("proj") or K1 ("fa"); plus the device timeline of "proj".
for cfg in "" "SPB_PACK_XH=0 SPB_XBAR_SCHED=proj" "SPB_PACK_XH=0 SPB_XBAR_SCHED=fa"; do
  for rep in 1 2; do
    env $cfg timeout 200 python bench.py --no-cpu > gpurun_out/x.json 2>/dev/null; echo "[$cfg] $(python tools/bench_summary.py gpurun_out/x.json 2>/dev/null | head -1)"
  done
done
SPB_PACK_XH=0 SPB_XBAR_SCHED=proj timeout 100 python tools/step_timeline.py 2>&1 | grep -v Warn
