# bench line's e2e leg only (device + host-link timing of the double-buffered requests)
timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"])'
