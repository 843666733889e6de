"""Chunk-length (T_c) sweep of the ALIF update (north_star (2)): for each
Tc, ms per update and the K6 carry kernel's time, algorithmic bytes and HBM fraction.

    python tools/tc_sweep.py [--hidden 1024] [--batch 256] [--T 2000] [--chunks 63,...,2047]

One JSON line per Tc.  K6 algorithmic bytes per launch = eps read (if loaded) + eps write
(if stored) + per-sample operands (W hi/lo 4 B and raw spikes 2 B per (b, rho, i|j)) +
the (M, Dt) coefficients; ncu DRAM bytes come from the profile capture beside it.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200.datasets import poisson_batch  # noqa: E402
from paper_2501_11407_b200.engine import EpropEngine, chunk_bytes  # noqa: E402
from paper_2501_11407_b200.gradients import _neuron_kwargs  # noqa: E402


def peaks():
    try:
        with open("MEASURED_PEAKS.json") as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hidden", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--T", type=int, default=2000)
    ap.add_argument("--chunks", default="63,127,255,511,1023,2047")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    n, B, T, k, m = args.hidden, args.batch, args.T, 700, 20
    hbm = peaks()
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f32", seed=0))
    kw = _neuron_kwargs(net)
    x, y = poisson_batch(B, k, T, m, seed=1)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for Tc in [int(c) for c in args.chunks.split(",")]:
        eng = EpropEngine(n, k, m, B, alif=True, chunk=Tc)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(xd, yd, binary=True, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            eng.run(xd, yd, binary=True, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        timers = {}
        eng.run(xd, yd, binary=True, timers=timers, **kw)
        torch.cuda.synchronize()
        carry_ms, carry_bytes, full = 0.0, 0.0, []
        eps = 4.0 * B * n * k
        for a, b, meta in timers.get("carry", []):
            ln, load, store, _raw = meta
            t = a.elapsed_time(b)
            byts = eps * (int(load) + int(store)) + 8.0 * B * n
            if store:   # the per-sample GEMM runs only when the trace is carried out
                byts += (4.0 * n + 2.0 * k) * B * (Tc + 1)
            carry_ms += t
            carry_bytes += byts
            if load and store:
                full.append(byts / (t * 1e-3) / 1e9 / hbm)
        row = {"Tc": Tc, "chunks": -(-T // Tc), "n_hidden": n, "batch": B, "T": T,
               "ms_per_update": ms, "samples_timesteps_per_s": B * T / (ms * 1e-3),
               "carry_ms_per_update": carry_ms,
               "carry_launches": len(timers.get("carry", [])),
               "carry_hbm_frac_all": (carry_bytes / (carry_ms * 1e-3) / 1e9 / hbm) if carry_ms else None,
               "carry_hbm_frac_full_launches": float(np.mean(full)) if full else None,
               "chunk_buffer_bytes": chunk_bytes(Tc, B, n, k),
               "hbm_peak_gbs": hbm}
        print(json.dumps(row), flush=True)
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
