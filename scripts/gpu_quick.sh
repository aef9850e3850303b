timeout 600 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "decode" 2>&1 | tail -2
for i in 1 2; do NOSTAMP=1 timeout 300 python scripts/dec_ts4.py 2>&1 | tail -1; done
timeout 300 python scripts/dec_ts4.py 2>&1 | grep -v Warn | grep "clk\|warp loop"
timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"], d["compress_ms_per_layer"])'
