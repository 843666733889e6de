# Multi-rank bench path on a 1-GPU box: two ranks share the GPU over gloo (not a
# performance number), weak and strong scaling; then the 1-rank line and the contract test.
mkdir -p gpurun_out/dist
export SPB_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/dist/dp2_weak.json 2> gpurun_out/dist/dp2_weak.err
echo "dp2 weak rc=$?"; tail -2 gpurun_out/dist/dp2_weak.err; python tools/bench_summary.py gpurun_out/dist/dp2_weak.json 2>/dev/null | head -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --gpus 2 --config c4 --global-batch 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/dist/dp2_strong.json 2> gpurun_out/dist/dp2_strong.err
echo "dp2 strong rc=$?"; tail -2 gpurun_out/dist/dp2_strong.err; python -c "
import json; d=json.loads(open('gpurun_out/dist/dp2_strong.json').read().strip().splitlines()[-1]); print(d['scaling'], d['config'], d['run']['launch'], d['value'], d['e2e']['value'])"
unset SPB_DIST_BACKEND
python bench.py --no-cpu > gpurun_out/dist/dp1.json 2>/dev/null; python tools/bench_summary.py gpurun_out/dist/dp1.json 2>/dev/null | head -1
timeout 900 python -m pytest tests/test_bench_contract.py tests/test_dist_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
