"""Benchmark of the B200 e-prop training step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Metric: e-prop train samples*timesteps/s on the SHD-shaped ALIF config (BASELINE.json
configs[2]: 700 -> 1024 ALIF -> 20, T=250, batch 256 per GPU), synthetic Poisson spikes
bit-identical to the reference generator, seeded reference initialisation.  One step
= one full e-prop update (pass A, readout/loss, pass B with all eligibility kernels,
gradient ready on device; for N>1 plus the single NCCL allreduce).  Weak scaling:
each rank processes its own batch of 256 samples.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
launching stream, with a 512 MiB L2 flush (> 126 MB L2) between timed steps outside
the events; barrier + synchronize on both sides; max over ranks.  ``e2e`` repeats the
step through the public engine API with pinned HOST inputs: H2D of the spike tensor
and labels and D2H of the per-sample losses are inside the timed region.

``--impl reference`` times the reference algorithm on the host CPU cores (the oracle
port, oracle/cpu_bench.py) on a bounded sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: kind, n, k, m, T, B (per GPU)
    "c2": ("lif", 256, 700, 20, 250, 128),
    "c3": ("alif", 1024, 700, 20, 250, 256),
    "c4": ("alif", 2048, 700, 35, 500, 128),
    "c5": ("alif", 1024, 700, 20, 2000, 256),
}
CONFIG_DESC = {
    "c2": "SHD-shaped LIF e-prop 700->256->20, T=250",
    "c3": "SHD-shaped ALIF e-prop 700->1024->20, T=250",
    "c4": "SSC-shaped ALIF e-prop 700->2048->35, T=500 (per-GPU shard of the 1024 batch at 8 GPUs)",
    "c5": "C5 sweep point: ALIF e-prop 700->1024->20, T=2000",
}
METRIC = "e-prop train samples·timesteps/s (SHD-shape ALIF); HBM GB/s vs roofline"
UNIT = "samples*timesteps/s"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


INT8_KERNELS = ("proj",)
# issue-rate peaks of the MMA kinds measured on this B200 (tools/mma_microbench.cu,
# profiles/r1/mma_microbench.txt: M = 128, N >= 128, one CTA per SM, burst clock)
MMA_ISSUE_PEAK_TOPS = {"proj": 4484.0, "gemm": 2196.0, "carry": 2196.0}


def measured_traffic(cfg, kernel):
    """DRAM bytes per launch (read + write) of ``kernel`` from the committed ncu capture of
    this config (profiles/*/traffic.json, tools/traffic_json.py), or None."""
    pdir = os.path.join(ROOT, "profiles")
    try:
        tags = sorted(d for d in os.listdir(pdir) if os.path.isdir(os.path.join(pdir, d)))
    except OSError:
        return None
    for tag in reversed(tags):
        try:
            with open(os.path.join(pdir, tag, "traffic.json")) as f:
                d = json.load(f)
            ent = d.get(cfg, {}).get(kernel)
            if ent:
                return {"bytes_per_launch": ent["bytes_per_launch"],
                        "source": f"profiles/{tag}/{ent['source']} (ncu, cold cache)"}
        except (OSError, ValueError):
            continue
    return None
FP32_PEAK_TFLOPS = 72.5  # FFMA/FFMA2 microbenchmark on this pool's B200 (tools/fp_microbench.cu)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# The W_out update runs after K7 on the engine's side stream, beside K5 (one rank):
# 0.6021 vs 0.6037 ms per update, e2e 106.2 vs 105.9 M (tools/wout_side_ab.sh, 3 alternating
# pairs).  SPB_WOUT_SIDE=0 puts it on the main stream at the end of the update (A/B).
WOUT_SIDE = os.environ.get("SPB_WOUT_SIDE", "1") != "0"


def parity_block(eng, net, x_np, y_np, kw, kind, recurrent=False):
    """One update of the timed configuration (the same engine, inputs and initial
    weights) checked against the f64 oracle -- the reference's BPTT engine batched in
    GEMM form (oracle/eprop_ref.bptt_batch, pinned to the reference's own outputs in
    tests/test_oracle.py).  Runs after the timed region; the oracle is only the checker.
    The full batch is checked when its [B, T, n] f64 oracle state fits 2^27 entries,
    else the first samples of the batch through a second engine of that size."""
    import torch
    from oracle import eprop_ref as O
    from paper_2501_11407_b200.engine import EpropEngine
    if recurrent:
        return {"checked": False, "why": "recurrent extension: parity unpinned (no reference)"}
    B, T, k = x_np.shape
    n = eng.n
    bs = B if B * T * n <= (1 << 27) else max(1, (1 << 27) // (T * n))
    e = eng
    if bs < B:
        e = EpropEngine(n, k, eng.m, bs, alif=kind == "alif", w_f64=False, chunk=eng.Tc,
                        device=eng.device)
    xs, ys = np.ascontiguousarray(x_np[:bs]), y_np[:bs]
    e.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    raster = torch.zeros((bs, T, (n + 31) // 32), dtype=torch.int32, device=eng.device)
    e.run(torch.from_numpy(xs).to(eng.device), torch.from_numpy(ys).to(eng.device),
          raster=raster, binary=True, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ref = O.bptt_batch(net.neuron.w, net.readout.w_out, O.Params(alif=kind == "alif"), xs, ys)
    t_or = time.perf_counter() - t0
    r = raster.cpu().numpy().view(np.uint32)
    got = ((r[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    got = got.reshape(bs, T, -1)[..., :n]
    gw = e.grad_w(torch.float64).cpu().numpy().ravel()
    gwo = e.grad_wout.cpu().numpy().ravel()
    rw, ro = ref.grad_w.ravel(), ref.grad_w_out.ravel()
    rel = float(np.linalg.norm(gw - rw) / np.linalg.norm(rw))
    cos = float(gw @ rw / (np.linalg.norm(gw) * np.linalg.norm(rw)))
    out = {
        "checked": True,
        "oracle": "f64 BPTT (reference gradients.py:188-231, batched GEMM form) on the "
                  "same inputs and initial weights",
        "samples": bs, "of_batch": B, "steps": T,
        "spike_flips": int((got != ref.raster).sum()),
        "spikes": int(ref.raster.sum()),
        "grad_w_rel_l2": rel, "grad_w_cos": cos,
        "grad_w_out_rel_l2": float(np.linalg.norm(gwo - ro) / np.linalg.norm(ro)),
        "loss_max_rel": float(np.max(np.abs(e.loss.cpu().numpy() - ref.loss)
                                     / np.maximum(np.abs(ref.loss), 1e-300))),
        "tolerance": "spikes bit-exact; grad rel <= 1e-4, cos >= 0.9999",
        "oracle_s": round(t_or, 2),
    }
    out["pass"] = bool(out["spike_flips"] == 0 and rel <= 1e-4 and cos >= 0.9999)
    return out


def dropin_e2e(P, net, x_np, y_np, chunk, calls=8):
    """The drop-in call a reference user makes, timed end to end on the host clock:
    ``eprop_batch_gradient(net, x, labels)`` with numpy uint8 spike counts in and numpy
    gradients out (and the same with bit-packed spikes, ``packed=True``).  Every call
    includes the host staging, the host-to-device input copy, the update and the
    device-to-host copies of the gradients, losses and readouts."""
    import torch
    from paper_2501_11407_b200.gradients import eprop_batch_gradient
    B, T, k = x_np.shape
    n, m = net.n, net.m
    out = {"input": "numpy uint8 spike counts [B, T, k]", "unit": UNIT}
    xb = np.packbits(x_np, axis=-1, bitorder="little")
    for tag, xin, kw in (("counts", x_np, {}), ("packed", xb, {"packed": True})):
        # eager, graph capture, replays -- until the pinned-host allocator caches two sets
        # of result buffers (the previous call's arrays are still alive during the next)
        for _ in range(4):
            r = eprop_batch_gradient(net, xin, y_np, chunk=chunk, **kw)
        torch.cuda.synchronize()
        per_call = []
        t0 = time.perf_counter()
        for _ in range(calls):
            t1 = time.perf_counter()
            r = eprop_batch_gradient(net, xin, y_np, chunk=chunk, **kw)
            per_call.append((time.perf_counter() - t1) * 1e3)
        dt = (time.perf_counter() - t0) / calls
        ent = {"value": B * T / dt, "ms_per_call": dt * 1e3,
               "ms_per_call_median": float(np.median(per_call)),
               "ms_per_call_each": [round(c, 3) for c in per_call],
               "h2d_bytes_per_call": int(xin.nbytes + y_np.nbytes),
               "d2h_bytes_per_call": int(4 * (n * k + m * n) + 8 * B + 8 * B * m + 4 * B)}
        if tag == "counts":
            from paper_2501_11407_b200.gradients import _staging, get_engine
            st = _staging(get_engine(net, B, chunk=chunk, T=T))
            ent["staging"] = "bytes (counts > 1)" if st.counts_nonbinary else \
                "bit-packed on the host (0/1 counts, spb_host_pack_bits)"
            out.update(ent)
        else:
            out["packed"] = dict(ent, input="np.packbits(x, axis=-1, bitorder='little')")
    out["calls"] = calls
    out["api"] = "paper_2501_11407_b200.eprop_batch_gradient (weights unchanged between calls)"
    del r
    return out


def shape_of(args, world):
    """(kind, n, k, m, T, B per rank, global batch, scaling) of the run: the config's
    per-GPU batch (weak scaling), or --global-batch split over the ranks (strong)."""
    kind, n, k, m, T, B = CONFIGS[args.config]
    n = getattr(args, "hidden", 0) or n          # C5 sweep points (--hidden / --seq-len)
    T = getattr(args, "seq_len", 0) or T
    if args.global_batch:
        if args.global_batch % world:
            raise SystemExit(f"--global-batch {args.global_batch} is not a multiple of {world}")
        return kind, n, k, m, T, args.global_batch // world, args.global_batch, "strong"
    return kind, n, k, m, T, B, B * world, "weak"


def config_dict(args, world, chunk):
    """The ``config`` object of the JSON line -- the same keys for both arms."""
    kind, n, k, m, T, B, G, scaling = shape_of(args, world)
    desc = CONFIG_DESC[args.config]
    if scaling == "strong":
        desc = desc.split(" (")[0] + f" (global batch {G} split over {world} rank(s))"
    if args.config == "c5":
        desc = f"C5 sweep point: ALIF e-prop 700->{n}->{m}, T={T}"
    return {"workload": desc + (" + recurrent W_rec" if args.recurrent else ""),
            "batch_per_gpu": B, "global_batch": G, "seq_len": T, "n_hidden": n,
            "n_inputs": k, "n_classes": m, "chunk": chunk, "parallelism": f"dp{world}"}


def cpu_reference_line(args, world):
    """--impl reference: the reference's own e-prop engine (ENGINES["eprop-sparse"],
    gradients.py:132-185, from baseline/_ref) on all host cores, rank 0 only; each timed
    step is a bounded sample of the workload (one T_sub-step sample per core)."""
    from oracle.cpu_bench import _pool, cores, cpu_model, reference_available, time_cpu, warm
    from paper_2501_11407_b200.engine import default_chunk
    kind, n, k, m, T, B, G, scaling = shape_of(args, world)
    impl = "reference" if reference_available() else "port"
    procs = cores()
    # bounded per-step sample: ~1 s of CPU work per timed step on this shape
    T_sub = max(2, min(T, int(25 * (1024 * 700) / (n * k)) if kind == "alif" else
                       int(100 * (256 * 700) / (n * k))))
    pool = _pool(procs)
    vals = []
    try:
        warm(pool, procs, kind, n, k, m, impl)
        for i in range(args.warmup + args.steps):
            v, wall, _ = time_cpu(kind, n, k, m, T_sub, procs, procs, pool=pool, impl=impl,
                                  warmed=True)
            if i >= args.warmup:
                vals.append(v)
    finally:
        pool.close()
        pool.join()
    value = float(np.mean(vals))
    what = ("the unmodified reference sparseprop 0.1.0 (baseline/_ref), "
            "ENGINES['eprop-sparse'] = gradients.py:132-185, f32 net"
            if impl == "reference" else
            "oracle port of gradients.py:132-185 (reference not installed in baseline/_ref)")
    sample = (f"{procs} processes x 1 sample x {T_sub} steps per timed step (of the "
              f"{G}x{T} workload); {what}; BLAS threads=1")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, world, default_chunk(T, B, n, k, kind == "alif")),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": impl,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--global-batch", type=int, default=0,
                    help="fixed global batch split over the ranks (strong scaling, e.g. "
                         "--config c4 --global-batch 1024); default: the config's batch "
                         "per GPU (weak scaling)")
    ap.add_argument("--chunk", type=int, default=0, help="0 = engine default for T")
    ap.add_argument("--hidden", type=int, default=0,
                    help="C5 sweep: hidden size override (BASELINE configs[4]: 256-8192)")
    ap.add_argument("--seq-len", type=int, default=0,
                    help="C5 sweep: sequence length override (BASELINE configs[4]: 100-10000)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-timing parity check of one update vs the f64 oracle")
    ap.add_argument("--park-gb", type=float, default=0.0,
                    help="opt-in: park every chunk's psi in pass A when it fits this many GB "
                         "(pass B skips the projection and dynamics; memory then grows with T)")
    ap.add_argument("--no-e2e-graph", dest="e2e_graph", action="store_false",
                    help="eager launches in the e2e loop (default: each step replays the "
                         "update's CUDA graph; measured 77-79 -> 79-81 M at C3)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="eager launches instead of replaying the captured CUDA graph")
    ap.add_argument("--recurrent", action="store_true",
                    help="recurrent W_rec extension (SURVEY.md 8(f)-4) on the chosen shape")
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu: no clocks, e2e or cpu baseline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_env()

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(cpu_reference_line(args, world)), flush=True)
        return

    import torch
    import torch.distributed as dist

    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200 import _lib
    from paper_2501_11407_b200.parallel import GradPacker

    # one GPU per rank (NCCL); SPB_DIST_BACKEND=gloo lets several ranks share one GPU to
    # exercise the multi-rank path (packing, allreduce, max over ranks) on a 1-GPU box
    backend = os.environ.get("SPB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    kind, n, k, m, T, B, G, scaling = shape_of(args, world)
    spec = P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m, precision="f32", seed=0,
                         recurrent=args.recurrent)
    net = P.init_network(spec)
    # this rank's shard: weak scaling -- its own batch (seed 1000 + rank); strong scaling
    # -- a contiguous slice of ONE global batch (seed 1000), every rank the same size
    if scaling == "strong":
        xg, yg = poisson_batch(G, k, T, m, seed=1000)
        x_np = np.ascontiguousarray(xg[rank * B:(rank + 1) * B])
        y_np = np.ascontiguousarray(yg[rank * B:(rank + 1) * B])
        del xg, yg
    else:
        x_np, y_np = poisson_batch(B, k, T, m, seed=1000 + rank)
    from paper_2501_11407_b200.engine import default_chunk
    chunk = args.chunk or default_chunk(T, B, n, k, kind == "alif")
    eng = EpropEngine(n, k, m, B, alif=kind == "alif", w_f64=False, chunk=chunk,
                      device=dev, recurrent=args.recurrent)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out),
                    w_rec=torch.from_numpy(net.neuron.w_rec) if args.recurrent else None)
    if args.park_gb > 0:
        eng.park_budget = int(args.park_gb * (1 << 30))
    xd = torch.from_numpy(x_np).to(dev)
    yd = torch.from_numpy(y_np).to(dev)
    # the payload: grad W columns [0, k) (+ grad W_rec columns [k, k + n), recurrent)
    kx = k + (n if args.recurrent else 0)
    packer = GradPacker(n, kx, m, dev)
    kw = dict(alpha=net.neuron.alpha, theta=net.neuron.theta, slope=net.neuron.slope,
              kappa=net.readout.kappa)
    if kind == "alif":
        kw.update(beta=net.neuron.beta, rho=net.neuron.rho)

    # Online weight update (north_star (3)): fp32 master W (the engine's) and W_out;
    # after the allreduce the fused SGD kernel updates both (W_out also refreshes the
    # engine's fp64 mirror) and W is re-sliced into the INT8 digits the next update's
    # projection reads -- all of it inside the timed step.
    wout_master = torch.from_numpy(np.ascontiguousarray(net.readout.w_out)).to(dev)
    wrec_master = (torch.from_numpy(np.ascontiguousarray(net.neuron.w_rec)).to(dev)
                   if args.recurrent else None)
    lr, g_scale = 1e-3, 1.0 / G
    vp = ctypes.c_void_p

    def update():
        if world > 1:  # the allreduced fp32 payload
            gw, gwo, _, _ = packer.views()
            g64, ldw = 0, kx
        else:          # one rank: straight from the engine's fp64 accumulators
            gw, gwo, g64, ldw = eng.grad_w_acc, eng.grad_wout, 1, eng.grad_w_acc.stride(0)
        main = torch.cuda.current_stream(dev)
        st = vp(main.cuda_stream)
        # W: SGD fused with the re-slicing of the first engine's INT8 digits
        eng.sgd_slice(gw, g64, ldw, g_scale, lr)
        # W_out: on one rank its gradient comes from K7 on the engine's side stream, so the
        # update follows K7 there (beside K5) and the step joins it at the end
        side = eng.side if (world == 1 and WOUT_SIDE) else None
        _lib.call("spb_sgd_update", vp(wout_master.data_ptr()), 0, m, n, vp(gwo.data_ptr()),
                  g64, n, g_scale, lr, vp(eng.wout.data_ptr()),
                  vp(side.cuda_stream) if side is not None else st)
        if side is not None:
            wo_done.record(side)
            main.wait_event(wo_done)
        if wrec_master is not None:  # W_rec (columns k .. k+n) and its transposed copy
            # (a small step size keeps the recurrent activity -- the gather work -- at its
            # initial level over the timed steps; at lr = 1e-3 the synthetic network's
            # recurrent excitation grows step by step.  Same kernels, same work per step.)
            _lib.call("spb_sgd_update", vp(wrec_master.data_ptr()), 0, n, n,
                      vp(gw.data_ptr() + gw.element_size() * k), g64, ldw, g_scale, 1e-6,
                      None, st)
            eng.wrecT.copy_(wrec_master.t())

    wo_done = torch.cuda.Event()

    def local_part(x, y, timers=None, bits=False):
        # the synthetic Poisson inputs are 0/1 spikes: promise it (K2 single-int64 path)
        eng.run(x, y, timers=timers, bits=bits, binary=True, **kw)
        if world > 1:
            packer.pack(eng.grad_w_acc, eng.grad_wout, eng.loss, eng.correct)

    def step(x, y, timers=None, bits=False):
        local_part(x, y, timers=timers, bits=bits)
        if world > 1:  # the update's single collective
            packer.allreduce()
        update()

    def captured_step(x, y, bits=False, loss_host=None):
        """The step as CUDA-graph replays on these input buffers: one graph at N = 1; at
        N > 1 the graph of the rank-local part (every kernel of the update and the payload
        pack), the allreduce launched eagerly on the same stream (collectives are not
        captured: a capture that succeeded on one rank but hung in replay on another would
        deadlock the job), then the graph of the optimizer step.  loss_host: the graph also
        copies the per-sample losses to this pinned host buffer, on a branch that follows
        the loss kernel (K3) and runs beside the rest of the update."""
        cs_ = torch.cuda.Stream(device=dev)
        cs_.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cs_):
            step(x, y, bits=bits)                   # warm the capture stream
        torch.cuda.current_stream(dev).wait_stream(cs_)
        g1 = torch.cuda.CUDAGraph()
        d2h = torch.cuda.Stream(device=dev) if loss_host is not None else None
        with torch.cuda.graph(g1, stream=cs_):
            local_part(x, y, bits=bits)
            if d2h is not None:
                ro = eng._ev.get("ro") if eng._ev else None
                if ro is not None:     # K3 done (recorded by run() for K7's side stream)
                    d2h.wait_event(ro)
                else:
                    d2h.wait_stream(cs_)
                with torch.cuda.stream(d2h):
                    loss_host.copy_(eng.loss, non_blocking=True)
                cs_.wait_stream(d2h)
            if world == 1:
                update()
        if world == 1:
            return g1.replay
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=cs_):
            update()

        def replay():
            g1.replay()
            packer.allreduce()
            g2.replay()
        return replay

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(xd, yd)
    barrier()

    # The whole update (every kernel, the side-stream fork/join, the gradient packing and
    # the allreduce) is captured once in a CUDA graph and replayed per step: no host
    # launch gaps on the device timeline.  Falls back to eager launches if capture fails.
    graph = None
    # N > 1: the rank-local part and the optimizer step are graphs, the allreduce between
    # them an eager collective (captured_step), so every N replays the same kernels.  All
    # ranks must agree on the mode.
    if args.graph and not args.profile:
        try:
            graph = captured_step(xd, yd)
            graph()
            barrier()
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] CUDA graph capture failed ({exc}); eager launches", file=sys.stderr)
            graph = None
            barrier()
        if world > 1:
            ok = torch.tensor([1 if graph is not None else 0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                graph = None

    clocks = ClockSampler(local) if not args.profile else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    timers = {}
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        if graph is not None:
            graph()
        else:
            step(xd, yd, timers=timers)
        ev[i][1].record()
    barrier()
    # kernels of libsparseprop_b200.so per step: the engine's + SGD(+slice) on W + SGD on
    # W_out (+ the payload pack when N > 1)
    launches_per_step = eng.launches + 2 + (1 if world > 1 else 0) + (1 if args.recurrent else 0)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    clk = clocks.stop() if clocks else None
    if graph is not None:  # per-kernel breakdown from eager steps (events per launch)
        n_bd = max(3, min(args.steps, 10))
        for _ in range(n_bd):
            flush.zero_()
            step(xd, yd, timers=timers)
        barrier()
    steps_bd = n_bd if graph is not None else args.steps

    # kernel breakdown (CUDA events on the launching stream)
    kern = {}
    for name, lst in timers.items():
        kern[name] = [(a.elapsed_time(b), meta) for a, b, meta in lst]

    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * B * T / (ms_max * 1e-3)

    # ---- e2e through the engine API with pinned host buffers ----
    # Each step's spikes/labels are copied H2D from pinned host memory on a copy stream
    # (double-buffered: step i+1's copy overlaps step i's kernels) and the per-sample
    # losses are read back D2H; every copy is inside the timed region.
    e2e = None
    if not args.no_e2e and not args.profile:
        # the host dataset holds the binary spike trains bit-packed (np.packbits, little
        # bit order): 1/8 of the uint8 bytes cross PCIe; K0 unpacks on the device
        x_bits = np.packbits(x_np, axis=-1, bitorder="little")
        xh = torch.from_numpy(x_bits).pin_memory()
        yh = torch.from_numpy(y_np).pin_memory()
        # the per-sample losses of step i go to pinned host memory: inside the replayed
        # graph on a branch after K3 (beside the rest of the update); eager steps stage them
        # on the device and read them back on the copy stream (double-buffered)
        loss_h = [torch.empty(B, dtype=torch.float64).pin_memory() for _ in range(2)]
        loss_s = [torch.empty(B, dtype=torch.float64, device=dev) for _ in range(2)]
        staged = [torch.cuda.Event() for _ in range(2)]
        read = [torch.cuda.Event() for _ in range(2)]
        xb = [torch.empty(x_bits.shape, dtype=torch.uint8, device=dev) for _ in range(2)]
        yb = [torch.empty_like(yd) for _ in range(2)]
        cs = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream(dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        for e in consumed + read:
            e.record(main)

        def prefetch(i):
            with torch.cuda.stream(cs):
                cs.wait_event(consumed[i % 2])
                xb[i % 2].copy_(xh, non_blocking=True)
                yb[i % 2].copy_(yh, non_blocking=True)
                copied[i % 2].record(cs)

        # one CUDA graph per input slot: the whole step (update included) on the double
        # buffer itself, replayed once its host-to-device copy has landed
        gsteps = None
        if args.e2e_graph and graph is not None:
            try:
                for i in range(2):
                    xb[i].copy_(torch.from_numpy(x_bits).to(dev))
                    yb[i].copy_(yd)
                torch.cuda.synchronize()
                gsteps = [captured_step(xb[i], yb[i], bits=True, loss_host=loss_h[i])
                          for i in range(2)]
                barrier()
            except Exception as exc:  # noqa: BLE001
                print(f"[bench] e2e graph capture failed ({exc}); eager", file=sys.stderr)
                gsteps = None

        def run_e2e(nsteps):
            prefetch(0)
            for i in range(nsteps):
                if i + 1 < nsteps:
                    prefetch(i + 1)
                main.wait_event(copied[i % 2])
                if gsteps is not None:
                    gsteps[i % 2]()
                else:
                    step(xb[i % 2], yb[i % 2], bits=True)
                consumed[i % 2].record(main)
                if gsteps is None:   # (the graph copies the losses itself)
                    main.wait_event(read[i % 2])
                    loss_s[i % 2].copy_(eng.loss, non_blocking=True)
                    staged[i % 2].record(main)
                    with torch.cuda.stream(cs):
                        cs.wait_event(staged[i % 2])
                        loss_h[i % 2].copy_(loss_s[i % 2], non_blocking=True)
                        read[i % 2].record(cs)
            main.wait_stream(cs)   # the last read-back is inside the timed region

        run_e2e(3)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        n_e2e = max(50, args.steps)   # short steps (C2) are host-jitter sensitive
        e0.record(main)
        run_e2e(n_e2e)
        e1.record(main)
        barrier()
        e2e_ms = torch.tensor([e0.elapsed_time(e1) / n_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": world * B * T / (float(e2e_ms.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(x_bits.nbytes + y_np.nbytes),
               "input_format": "bit-packed binary spikes (np.packbits, little), unpacked on device",
               "d2h_bytes_per_step": int(B * 8),
               "ms_per_step": float(e2e_ms.item()),
               "pipeline": "H2D of step i+1 on a copy stream overlaps step i (double buffer); "
                           "step i's losses are copied D2H right after its loss kernel, beside "
                           "the rest of the update"
                           + ("; each step replays the whole update's CUDA graph"
                              if gsteps is not None else "")}

    # ---- roofline of every main kernel; the dominant one is the headline ----
    hbm_peak, bf16_peak, peak_kind = peaks()
    Tc, KR, P_sl = eng.Tc, eng.KR, eng.P
    kernels = {}
    for name, lst in kern.items():
        t_tot = sum(t for t, _ in lst) * 1e-3                    # seconds over all steps
        byts = flops = 0.0
        for _, meta in lst:
            if name == "proj":
                ln = meta                                        # int8 MACs x2, useful part
                flops += 2.0 * P_sl * B * ln * n * k
                byts += B * ln * k + P_sl * n * k + 8.0 * B * ln * n
            elif name in ("forward", "forward_a"):
                ln, pid, flag = meta
                pid = {3: 2, 4: 1}.get(pid, pid)   # raw-operand passes: same traffic
                psi = 4.0 * B * (ln + 1) * n
                if pid <= 1:                       # dynamics: read the fp64 current
                    byts += 8.0 * B * ln * n
                    if pid == 1 or flag:           # psi parked for the scan
                        byts += psi
                if pid >= 1:                       # scan: psi back, C (and W) out, bf16 hi/lo
                    byts += psi + 4.0 * n * B * KR * (2 if flag else 1)
            elif name == "gemm":
                ln, raw = meta                   # raw spikes (exact bf16): 2 MMAs, no B-lo
                flops += (4.0 if raw else 6.0) * n * k * B * (ln + 1)
                byts += 4.0 * n * B * KR + (2.0 if raw else 4.0) * k * B * KR
            elif name == "carry":
                ln, ld, stv, raw = meta             # raw spikes: 2 MMAs, x hi only (2 B)
                byts += 4.0 * B * n * k * (int(ld) + int(stv)) + 8.0 * B * n
                if stv:
                    byts += (4.0 * n + (2.0 if raw else 4.0) * k) * B * KR
                    flops += (4.0 if raw else 6.0) * n * k * B * KR
        ent = {"ms_per_step": t_tot * 1e3 / steps_bd, "share_of_step": t_tot * 1e3 / steps_bd / ms,
               "launches_per_step": len(lst) / steps_bd}
        if byts:
            ent["hbm_gbs"] = byts / t_tot / 1e9
            ent["hbm_frac"] = ent["hbm_gbs"] / hbm_peak
        if flops:
            pk = 2 * bf16_peak if name in INT8_KERNELS else bf16_peak
            ent["tensor_tflops"] = flops / t_tot / 1e12
            ent["tensor_frac"] = ent["tensor_tflops"] / pk
        kernels[name] = ent
    roof = None
    if kernels:
        dom = max(kernels, key=lambda nm: kernels[nm]["ms_per_step"])
        e = kernels[dom]
        names = {"proj": "input_proj_kernel (K2, int8 tcgen05)", "forward": "forward_chunk + chunk_scan (K1 pass B)",
                 "forward_a": "forward_chunk_kernel (K1 pass A)",
                 "gemm": "grad_gemm_tc_kernel (K5, bf16 hi/lo tcgen05)",
                 "carry": "alif_carry_pair_kernel (K6p, cta_group::2 tcgen05 + eps stream)"}
        if args.recurrent:
            names["forward_a"] = "forward_rec_kernel (K1rec pass A: recurrent spike gather)"
        if e.get("tensor_frac", 0) >= e.get("hbm_frac", 0) and "tensor_tflops" in e:
            pk = 2 * bf16_peak if dom in INT8_KERNELS else bf16_peak
            roof = {"kernel": names[dom], "bound": "tensor", "achieved": e["tensor_tflops"],
                    "peak": pk, "unit": "TFLOP/s", "frac": e["tensor_frac"]}
        else:
            roof = {"kernel": names[dom], "bound": "hbm", "achieved": e["hbm_gbs"],
                    "peak": hbm_peak, "unit": "GB/s", "frac": e["hbm_frac"]}
        tr = measured_traffic(args.config + ("_rec" if args.recurrent else ""), dom)
        if roof["bound"] == "tensor" and dom in MMA_ISSUE_PEAK_TOPS:
            # the same achieved rate against the MMA kind's own measured issue peak
            roof["frac_of_mma_issue_peak"] = roof["achieved"] / MMA_ISSUE_PEAK_TOPS[dom]
            roof["mma_issue_peak_source"] = ("tools/mma_microbench.cu "
                                             "(profiles/r1/mma_microbench.txt), burst clock")
        roof.update({"peak_source": peak_kind + (" (int8 = 2x bf16)" if dom in INT8_KERNELS else ""),
                     "traffic": (tr or {}).get("bytes_per_launch"),
                     "traffic_unit": "bytes per launch (DRAM read + write)",
                     "traffic_source": (tr or {}).get("source"),
                     "kernel_ms_per_step": e["ms_per_step"],
                     "share_of_step": e["share_of_step"]})

    # ---- drop-in API end to end (rank 0, N=1): eprop_batch_gradient on numpy ----
    # (before the parity oracle and the CPU arm: their numpy / BLAS threads would compete
    # with the drop-in's host staging threads)
    dropin = None
    if world == 1 and not args.no_e2e and not args.profile and not args.recurrent:
        dropin = dropin_e2e(P, net, x_np, y_np, chunk)

    # ---- parity of the timed configuration (after the timed region; rank 0) ----
    parity = None
    if rank == 0 and not args.no_parity and not args.profile:
        try:
            parity = parity_block(eng, net, x_np, y_np, kw, kind, args.recurrent)
        except Exception as exc:  # noqa: BLE001
            parity = {"checked": False, "error": repr(exc)}

    # ---- CPU baseline (rank 0, N=1 only) ----
    # the reference's own engine (baseline/_ref) is the baseline; the oracle port of the
    # same algorithm is reported beside it, labelled
    cpu = cpu_port = None
    if world == 1 and not args.no_cpu and not args.profile:
        from oracle.cpu_bench import cores, cpu_model, reference_available, time_cpu
        procs = cores()
        for impl in (("reference", "port") if reference_available() else ("port",)):
            per_core = 10 if impl == "reference" else 40      # bounded: ~5-10 s each
            T_sub = max(2, min(T, int(per_core * (1024 * 700) / (n * k)) if kind == "alif"
                               else int(4 * per_core * (256 * 700) / (n * k))))
            v, wall, procs = time_cpu(kind, n, k, m, T_sub, 2 * procs, procs, impl=impl)
            what = ("the unmodified reference sparseprop 0.1.0 (baseline/_ref), "
                    "ENGINES['eprop-sparse'], f32 net" if impl == "reference" else
                    "oracle port (oracle/eprop_ref.eprop_forward_mode) of gradients.py:132-185")
            ent = {"value": v, "unit": UNIT, "cores": procs, "kind": impl,
                   "cpu_model": cpu_model(),
                   "sample": f"{2 * procs} single-sample tasks x {T_sub} steps of the "
                             f"{B}x{T} workload on {procs} processes ({wall:.1f} s wall); "
                             f"{what}; BLAS threads=1"}
            if impl == "reference" or cpu is None:
                cpu = ent
            if impl == "port":
                cpu_port = ent

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, world, eng.Tc),
            "run": {"forward_precision": "fp64 state/current (bit-exact spikes)",
                    "forward_kernel": "K2 projection + K1 dynamics",
                    "step": "e-prop gradient (+ allreduce when N > 1) + fused SGD on W/W_out "
                            "+ W re-slice" + (" + SGD on W_rec (+ its transposed copy)"
                                              if args.recurrent else ""),
                    "psi_parking_gb": args.park_gb,
                    "l2": "512 MiB flush between timed steps (outside events)",
                    "launch": (("CUDA graph replay of the whole update" if world == 1 else
                                "CUDA graph replays of the rank-local update and of the "
                                "optimizer step around one eager allreduce")
                               if graph is not None else "eager launches"),
                    "dist_backend": backend if world > 1 else None},
            "memory": {"engine_device_bytes": eng.device_bytes(),
                       "peak_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
                       "note": "engine_device_bytes = every buffer of the update (sized by "
                               "B, n, k and the chunk, not by T); the peak also holds the "
                               "device-resident input batch [B, T, k] and the L2 flush buffer"},
            "e2e": e2e,
            "e2e_dropin": dropin,
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "cpu_baseline_port": cpu_port,
            "parity": parity,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
