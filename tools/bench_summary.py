import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith("{"): print(line); continue
    d=json.loads(line)
    print("chunk", d["config"]["chunk"], "ms", round(d["ms_per_step"],3), "value %.3g"%d["value"])
    for k,v in d["kernels"].items(): print("   ", k, {a: round(b,3) for a,b in v.items()})
    print("   roof", d["roofline"])
