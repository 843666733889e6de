"""Top SASS instructions of an ncu report (source page): by warp-stall samples and by
executed instructions; plus the opcode mix of the executed instructions."""
import collections, csv, io, subprocess, sys


def main(path, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hi = his[0]  # first kernel of the report (a report may hold several launches)
    hdr = rows[hi]
    end = his[1] if len(his) > 1 else len(rows)
    data = [r for r in rows[hi + 1:end] if len(r) == len(hdr) and r[0] != "Address"]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    val = lambda r, i: float(r[i]) if r[i] not in ("", "-") else 0.0
    tot = sum(val(r, si) for r in data) or 1.0
    etot = sum(val(r, ei) for r in data) or 1.0
    print(f"{path}: {int(tot)} stall samples, {int(etot)} warp instructions")
    for r in sorted(data, key=lambda r: -val(r, si))[:top]:
        print(f"{100*val(r, si)/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
    mix = collections.Counter()
    for r in data:
        op = r[1].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        mix[o.split(".")[0]] += val(r, ei)
    print("opcode mix (executed):")
    for o, c in mix.most_common(20):
        print(f"  {o:12s} {100*c/etot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
