"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel (shares)."""
import collections, csv, sys

def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi:
            continue
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")) * scale[r[ui]])
    tot = sum(sum(v) for v in agg.values())
    print(f"{'us total':>10} {'launches':>8} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v):10.1f} {len(v):8d} {100*sum(v)/tot:5.1f}%  {k}")

if __name__ == "__main__":
    main(sys.argv[1])
