"""C5 sweep (BASELINE.json configs[4]): ALIF hidden 256-8192 x T 100-10000 at a fixed batch
(B = 256).  Each point is one `bench.py --config c5 --hidden n --seq-len T` run (CUDA-graph
update, per-kernel CUDA events, memory); this prints one summary line per point plus the
flatness of the engine's device memory in T per hidden size.

    python tools/c5_sweep.py [--hidden 256,1024,4096,8192] [--T 100,1000,10000] [--batch 256]
                             [--parity-max-n 256] [--out gpurun_out/c5/sweep.jsonl]

Parity (the bench's f64-oracle check of one update on a sample subset) runs for hidden
sizes <= --parity-max-n.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hidden", default="256,1024,4096,8192")
    ap.add_argument("--T", default="100,1000,10000")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--parity-max-n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5", "sweep.jsonl"))
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    rows = []
    with open(args.out, "w") as fo:
        for n in [int(v) for v in args.hidden.split(",")]:
            per_n = []
            for T in [int(v) for v in args.T.split(",")]:
                cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5",
                       "--hidden", str(n), "--seq-len", str(T), "--global-batch",
                       str(args.batch), "--steps", str(args.steps), "--warmup", "3",
                       "--no-e2e", "--no-cpu"]
                if n > args.parity_max_n:
                    cmd.append("--no-parity")
                p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
                line = None
                for ln in p.stdout.splitlines():
                    if ln.startswith("{"):
                        line = json.loads(ln)
                if line is None:
                    row = {"n_hidden": n, "T": T, "error": p.stderr[-600:]}
                else:
                    k = line["kernels"]
                    carry = k.get("carry", {})
                    par = line.get("parity") or {}
                    row = {"n_hidden": n, "T": T, "batch": args.batch,
                           "chunk": line["config"]["chunk"],
                           "samples_timesteps_per_s": line["value"],
                           "ms_per_update": line["ms_per_step"],
                           "dominant_kernel": line["roofline"]["kernel"],
                           "dominant_bound": line["roofline"]["bound"],
                           "dominant_frac": line["roofline"]["frac"],
                           "kernel_share": {nm: round(e["share_of_step"], 3)
                                            for nm, e in k.items()},
                           "kernel_frac": {nm: round(e.get("tensor_frac", e.get("hbm_frac", 0)), 3)
                                           for nm, e in k.items()},
                           "carry_hbm_frac": carry.get("hbm_frac"),
                           "engine_device_bytes": line["memory"]["engine_device_bytes"],
                           "peak_allocated_bytes": line["memory"]["peak_allocated_bytes"],
                           "parity": ({"samples": par.get("samples"),
                                       "spike_flips": par.get("spike_flips"),
                                       "grad_w_rel_l2": par.get("grad_w_rel_l2"),
                                       "grad_w_cos": par.get("grad_w_cos"),
                                       "pass": par.get("pass")}
                                      if par.get("checked") else None),
                           "clocks": line.get("clocks")}
                print(json.dumps(row), flush=True)
                fo.write(json.dumps(row) + "\n")
                fo.flush()
                per_n.append(row)
            ok = [r for r in per_n if "engine_device_bytes" in r]
            if ok:
                # memory must not grow with T: the engine at ONE chunk length (the one the
                # longest T gets) for every T -- buffers are sized by (B, n, k, chunk) only
                chunk = ok[-1]["chunk"]
                mem = {}
                for T in [int(v) for v in args.T.split(",")]:
                    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5",
                           "--hidden", str(n), "--seq-len", str(T), "--global-batch",
                           str(args.batch), "--chunk", str(chunk), "--steps", "3",
                           "--warmup", "3", "--no-e2e", "--no-cpu", "--no-parity"]
                    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
                    for ln in p.stdout.splitlines():
                        if ln.startswith("{"):
                            d = json.loads(ln)
                            mem[T] = {"engine_device_bytes": d["memory"]["engine_device_bytes"],
                                      "ms_per_update": d["ms_per_step"]}
                vals = [v["engine_device_bytes"] for v in mem.values()]
                summ = {"n_hidden": n, "fixed_chunk": chunk, "by_T": mem,
                        "engine_bytes_max_over_min": (max(vals) / min(vals)) if vals else None}
                print(json.dumps(summ), flush=True)
                fo.write(json.dumps(summ) + "\n")
            rows.extend(per_n)


if __name__ == "__main__":
    main()
