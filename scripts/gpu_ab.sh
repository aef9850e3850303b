for cs in 6 7 10; do
export ADAKV_DECODE_CS=$cs
echo "cs $cs $(timeout 900 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])')"
done
