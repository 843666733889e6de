# A/B of the W_out update's placement at C3: after K7 on the side stream, beside K5
# (default) vs on the main stream at the end of the update (SPB_WOUT_SIDE=0) -- device timelines
for f in "" "--no-side"; do
  echo "== step_timeline $f"
  timeout 100 python tools/step_timeline.py $f 2>&1 | grep -v -i warn | tail -6
done
