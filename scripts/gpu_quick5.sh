timeout 800 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "decode" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])'; done
