"""C5 sweep (BASELINE.json configs[4]): ALIF hidden 256-8192, T 100-10000 at fixed batch,
streamed inputs -- peak device memory vs T (must be flat) and throughput.

    python tools/mem_sweep.py [--batch 64] [--hidden 256,1024,4096,8192] [--T 100,1000,10000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200.datasets import poisson_batch  # noqa: E402
from paper_2501_11407_b200.engine import EpropEngine  # noqa: E402
from paper_2501_11407_b200.gradients import _neuron_kwargs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--hidden", default="256,1024,4096,8192")
    ap.add_argument("--T", default="100,1000,10000")
    ap.add_argument("--chunk", type=int, default=0, help="0 = engine default (memory-budgeted)")
    args = ap.parse_args()
    B, k, m = args.batch, 700, 20
    for n in [int(v) for v in args.hidden.split(",")]:
        net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=m,
                                           precision="f32", seed=0))
        kw = _neuron_kwargs(net)
        rows = []
        Ts = [int(v) for v in args.T.split(",")]
        from paper_2501_11407_b200.engine import default_chunk
        # one chunk length for the whole sweep (the one the longest T gets), so the
        # footprint comparison is across T only
        chunk = args.chunk or default_chunk(max(Ts), B, n, k)
        for T in Ts:
            x, y = poisson_batch(B, k, T, m, seed=1)
            xh = torch.from_numpy(x).pin_memory()
            yd = torch.from_numpy(y).cuda()
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            torch.cuda.reset_peak_memory_stats()
            base = torch.cuda.memory_allocated()
            eng = EpropEngine(n, k, m, B, alif=True, chunk=chunk)
            eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
            eng.run(xh, yd, **kw)                      # warm-up
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 3
            for _ in range(reps):
                eng.run(xh, yd, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            peak = torch.cuda.max_memory_allocated() - base
            rows.append({"n_hidden": n, "T": T, "batch": B, "chunk": chunk,
                         "peak_device_bytes": int(peak),
                         "ms_per_update": ms, "samples_timesteps_per_s": B * T / (ms * 1e-3),
                         "inputs": "streamed from pinned host memory (H2D inside the timing)"})
            del eng
        ratio = rows[-1]["peak_device_bytes"] / rows[0]["peak_device_bytes"]
        for r in rows:
            r["peak_ratio_vs_shortest_T"] = r["peak_device_bytes"] / rows[0]["peak_device_bytes"]
            print(json.dumps(r), flush=True)
        print(json.dumps({"n_hidden": n, "peak_T_ratio": ratio, "flat": ratio <= 1.05}), flush=True)


if __name__ == "__main__":
    main()
