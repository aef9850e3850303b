for r in 1 2; do echo "run $(timeout 900 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])' 2>&1)"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k decode 2>&1 | tail -1
