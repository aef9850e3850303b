for r in 1 2; do
echo "mma.sync $(timeout 900 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])' 2>&1)"
echo "umma     $(ADAKV_DECODE_UMMA=1 timeout 900 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])' 2>&1)"
done
ADAKV_DECODE_UMMA=1 timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
