mkdir -p gpurun_out/r2b
timeout 600 python bench.py > gpurun_out/r2b/bench_c3.json 2> gpurun_out/r2b/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu --steps 10 > gpurun_out/r2b/bench_c4.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > gpurun_out/r2b/bench_c2.json 2>&1
for c in c3 c4 c2; do python -c "import json; d=json.loads(open('gpurun_out/r2b/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['e2e']['value'], d['e2e_dropin']['ms_per_call'], d['e2e_dropin']['packed']['ms_per_call'])"; done
