python tools/passb_check.py
for c in c3 c4 c2; do for g in 1 2 3 4; do SPB_PASSB_GROUPS=$g timeout 300 python bench.py --config $c --no-cpu --steps 30 > gpurun_out/ab.json 2>/dev/null; echo -n "$c G=$g "; python tools/bench_summary.py gpurun_out/ab.json 2>/dev/null | grep -E "ms=" | sed -E 's/.*ms=([0-9.]+).*/ms=\1/'; done; done
