"""Compact summary of bench.py JSON lines (files given as arguments, or stdin)."""
import json
import sys


def show(d):
    c = d["config"]
    print(f"{c['workload'][:40]} B={c['batch_per_gpu']} T={c['seq_len']} chunk={c['chunk']} "
          f"ms={d['ms_per_step']:.4f} value={d['value']:.4g} e2e={(d.get('e2e') or {}).get('value', 0):.4g}")
    for k, v in (d.get("kernels") or {}).items():
        print("   ", k, {a: round(b, 3) for a, b in v.items()})
    r = d.get("roofline") or {}
    print("    roofline", {k: r.get(k) for k in ("kernel", "bound", "frac")})
    if d.get("parity"):
        p = d["parity"]
        print("    parity", {k: p.get(k) for k in ("pass", "spike_flips", "grad_w_rel_l2")})
    if d.get("e2e_dropin"):
        e = d["e2e_dropin"]
        print("    dropin ms/call", round(e["ms_per_call"], 3), "packed", round(e["packed"]["ms_per_call"], 3))


srcs = [open(p) for p in sys.argv[1:]] or [sys.stdin]
for f in srcs:
    for line in f:
        line = line.strip()
        if line.startswith("{"):
            show(json.loads(line))
