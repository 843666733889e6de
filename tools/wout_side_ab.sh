# A/B of bench.py's SPB_WOUT_SIDE (W_out update beside K5 on the side stream vs at the end of
# the update on the main stream): device ms/update and the e2e loop, alternating, 3 reps
for rep in 1 2 3; do for v in 1 0; do
  SPB_WOUT_SIDE=$v timeout 200 python bench.py --no-cpu --no-parity --steps 30 > gpurun_out/e.json 2>/dev/null; echo "side=$v $(python tools/bench_summary.py gpurun_out/e.json 2>/dev/null | head -1)"
done; done
