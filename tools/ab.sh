# A/B of library variants built by tools/build_variant.sh:  bash tools/ab.sh <variant> [configs]
V=${1:-elect}
mkdir -p gpurun_out
for L in "" ab/lib_$V.so; do echo "== lib ${L:-default}"; SPB_LIB=$L timeout 120 python tools/proj_probe.py 2>&1 | grep -E "probe=0 |probe=3 |probe=39 \{\}|probe=36 \{\}"; done
SPB_LIB=ab/lib_$V.so timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "projection or banded or int8" 2>&1 | tail -1
for rep in 1 2; do for L in "" ab/lib_$V.so; do
  SPB_LIB=$L timeout 180 python bench.py --no-cpu > gpurun_out/ab.json 2>/dev/null; python tools/bench_summary.py gpurun_out/ab.json | head -1 | sed "s|^|${L:-default} |"
done; done
