"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernels
captured by tools/capture_profiles.sh, keyed by bench config and bench kernel name, for
bench.py's roofline.traffic.  Usage: python tools/traffic_json.py <gpurun_out/tag> > traffic.json"""
import csv, io, json, os, subprocess, sys

# ncu capture -> (bench config, bench kernel name)
CAPTURES = {
    "ncu_input_proj": ("c3", "proj"),
    "ncu_forward_chunk": ("c3", "forward_a"),
    "ncu_chunk_scan": ("c3", "forward"),
    "ncu_grad_gemm": ("c3", "gemm"),
    "ncu_xbar_chunk": ("c3", "xbar"),
    "ncu_alif_carry": ("c5", "carry"),
    "ncu_alif_carry_tc511": ("c5", "carry"),
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(src):
    out = {}
    for stem, (cfg, name) in CAPTURES.items():
        path = os.path.join(src, stem + ".ncu-rep")
        if not os.path.exists(path):
            continue
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        vals = []
        for r in rows[2:]:
            tot = 0.0
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(key)
                tot += float(r[i].replace(",", "")) * SCALE[units[i]]
            vals.append(tot)
        if vals:
            out.setdefault(cfg, {})[name] = {"bytes_per_launch": sum(vals) / len(vals),
                                             "launches": len(vals), "source": stem + ".ncu-rep"}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
