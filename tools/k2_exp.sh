timeout 300 python bench.py --recurrent --no-cpu --steps 10 > gpurun_out/r2b/bench_c3_recurrent.json 2>gpurun_out/r2b/rec.err; tail -2 gpurun_out/r2b/rec.err
python tools/bench_summary.py gpurun_out/r2b/bench_c3_recurrent.json | head -3
SPB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --recurrent --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-200
