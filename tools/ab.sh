for L in base nofence; do echo "== $L"; SPB_LIB=ab/lib_$L.so python tools/proj_probe.py 2>&1 | grep -E "probe=0 |probe=3 |probe=39 \{\}|probe=36"; done
SPB_LIB=ab/lib_nofence.so timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "projection or banded or int8" 2>&1 | tail -1
