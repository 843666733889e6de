"""Device timeline of the C3 update as the bench replays it (one CUDA graph per update):
per-kernel start/end from CUPTI (torch.profiler), averaged over several replays, with the
idle gaps between consecutive kernels -- where the ms/update goes.
    python tools/step_timeline.py [--config c3] [--replays 10]"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2501_11407_b200 as P
from paper_2501_11407_b200 import _lib
from paper_2501_11407_b200.datasets import poisson_batch
from paper_2501_11407_b200.engine import EpropEngine, default_chunk

ap = argparse.ArgumentParser()
ap.add_argument("--replays", type=int, default=10)
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--T", type=int, default=250)
ap.add_argument("--out", default="gpurun_out/step_timeline.json")
ap.add_argument("--no-side", dest="side", action="store_false",
                help="W_out update on the main stream (bench.py SPB_WOUT_SIDE=0)")
args = ap.parse_args()

n, k, m, T, B = 1024, 700, 20, args.T, args.B
dev = torch.device("cuda", 0)
net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=m,
                                   precision="f32", seed=0))
x_np, y_np = poisson_batch(B, k, T, m, seed=1000)
eng = EpropEngine(n, k, m, B, alif=True, w_f64=False, chunk=default_chunk(T, B, n, k, True),
                  device=dev)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
xd, yd = torch.from_numpy(x_np).to(dev), torch.from_numpy(y_np).to(dev)
wout = torch.from_numpy(np.ascontiguousarray(net.readout.w_out)).to(dev)
kw = dict(alpha=net.neuron.alpha, theta=net.neuron.theta, slope=net.neuron.slope,
          kappa=net.readout.kappa, beta=net.neuron.beta, rho=net.neuron.rho)
vp = ctypes.c_void_p


wo_done = torch.cuda.Event()


def step():  # as bench.py's update at one rank
    eng.run(xd, yd, binary=True, **kw)
    main = torch.cuda.current_stream(dev)
    st = vp(main.cuda_stream)
    eng.sgd_slice(eng.grad_w_acc, 1, eng.grad_w_acc.stride(0), 1.0 / B, 1e-3)
    side = eng.side if args.side else None
    _lib.call("spb_sgd_update", vp(wout.data_ptr()), 0, m, n, vp(eng.grad_wout.data_ptr()), 1,
              n, 1.0 / B, 1e-3, vp(eng.wout.data_ptr()),
              vp(side.cuda_stream) if side is not None else st)
    if side is not None:
        wo_done.record(side)
        main.wait_event(wo_done)


cs = torch.cuda.Stream(device=dev)
cs.wait_stream(torch.cuda.current_stream(dev))
with torch.cuda.stream(cs):
    for _ in range(3):
        step()
torch.cuda.current_stream(dev).wait_stream(cs)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=cs):
    step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(args.replays):
        flush.zero_()
        g.replay()
    torch.cuda.synchronize()
path = "/tmp/step_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"]
      if e.get("cat") == "kernel" and "FillFunctor" not in e.get("name", "")]
ev.sort(key=lambda e: e["ts"])
# split into replays: the first kernel of every update is the spike pack
steps, cur = [], []
first = ev[0]["name"]
for e in ev:
    if e["name"] == first and cur:
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
steps = [s for s in steps if len(s) == len(steps[-1])][1:]  # drop the first (cold) replay
rows = []
nk = len(steps[0])
for i in range(nk):
    dur = [s[i]["dur"] for s in steps]
    start = [s[i]["ts"] - s[0]["ts"] for s in steps]
    end = [s[i]["ts"] + s[i]["dur"] - s[0]["ts"] for s in steps]
    rows.append(dict(kernel=steps[0][i]["name"][:60], stream=steps[0][i].get("tid"),
                     start_us=float(np.median(start)), dur_us=float(np.median(dur)),
                     end_us=float(np.median(end))))
span = float(np.median([s[-1]["ts"] + s[-1]["dur"] - s[0]["ts"] for s in steps]))
last_end = 0.0
print(f"{'start':>8} {'dur':>8} {'gap':>6}  stream  kernel")
for r in rows:
    gap = r["start_us"] - last_end
    print(f"{r['start_us']:8.1f} {r['dur_us']:8.1f} {gap:6.1f}  {r['stream']!s:>6}  {r['kernel']}")
    last_end = max(last_end, r["end_us"])
print(f"update span (first kernel start -> last kernel end): {span:.1f} us over {len(steps)} replays")
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(dict(rows=rows, span_us=span, replays=len(steps)), open(args.out, "w"), indent=1)
