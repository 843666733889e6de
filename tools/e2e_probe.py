"""Where the e2e loop's time goes at C3: graph replays back to back (no copies), + the
H2D of bit-packed spikes on a copy stream, + the per-step loss D2H on the main stream,
+ the D2H moved to a side stream from a device staging copy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200.datasets import poisson_batch  # noqa: E402
from paper_2501_11407_b200.engine import EpropEngine  # noqa: E402
from paper_2501_11407_b200.gradients import _neuron_kwargs  # noqa: E402

n, k, m, T, B = 1024, 700, 20, 250, 256
net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=m,
                                   precision="f32", seed=0))
kw = _neuron_kwargs(net)
x, y = poisson_batch(B, k, T, m, seed=1000)
xbits = np.packbits(x, axis=-1, bitorder="little")
xh = torch.from_numpy(xbits).pin_memory()
yh = torch.from_numpy(y).pin_memory()
eng = EpropEngine(n, k, m, B, alif=True, chunk=255)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
xb = [torch.from_numpy(xbits).cuda() for _ in range(2)]
yb = [torch.from_numpy(y).cuda() for _ in range(2)]
steps = [eng.graphed(xb[i], yb[i], static_inputs=True, bits=True, binary=True, **kw)
         for i in range(2)]
main = torch.cuda.current_stream()
cs = torch.cuda.Stream()
ds = torch.cuda.Stream()
loss_h = [torch.empty(B, dtype=torch.float64).pin_memory() for _ in range(2)]
loss_d = [torch.empty(B, dtype=torch.float64, device="cuda") for _ in range(2)]
copied = [torch.cuda.Event() for _ in range(2)]
consumed = [torch.cuda.Event() for _ in range(2)]
done = [torch.cuda.Event() for _ in range(2)]
for e in consumed:
    e.record(main)


def prefetch(i):
    with torch.cuda.stream(cs):
        cs.wait_event(consumed[i % 2])
        xb[i % 2].copy_(xh, non_blocking=True)
        yb[i % 2].copy_(yh, non_blocking=True)
        copied[i % 2].record(cs)


def run(mode, N):
    if mode != "replay":
        prefetch(0)
    for i in range(N):
        if mode != "replay":
            if i + 1 < N:
                prefetch(i + 1)
            main.wait_event(copied[i % 2])
        steps[i % 2]()
        consumed[i % 2].record(main)
        if mode == "d2h_main":
            loss_h[0].copy_(eng.loss, non_blocking=True)
        elif mode == "d2h_side":
            loss_d[i % 2].copy_(eng.loss, non_blocking=True)   # D2D on main (tiny)
            done[i % 2].record(main)
            with torch.cuda.stream(ds):
                ds.wait_event(done[i % 2])
                loss_h[i % 2].copy_(loss_d[i % 2], non_blocking=True)


for mode in ("replay", "h2d", "d2h_main", "d2h_side", "replay"):
    run(mode, 5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N = 30
    a.record(main)
    run(mode, N)
    b.record(main)
    torch.cuda.synchronize()
    print(mode, "ms/step", round(a.elapsed_time(b) / N, 4), flush=True)
