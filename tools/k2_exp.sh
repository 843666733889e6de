timeout 600 python bench.py --no-cpu --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e_dropin'])"
