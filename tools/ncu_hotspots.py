"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, io, subprocess, sys

def main(path, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[si]) for r in data) or 1.0
    data.sort(key=lambda r: -float(r[si]))
    print(f"{path}: {int(tot)} samples")
    for r in data[:top]:
        print(f"{100*float(r[si])/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
