# decode launch-shape sweep on the bench (env overrides), interleaved
for r in 1 2; do for cfg in "CS=9" "CS=8" "CS=7" "CS=10"; do
  cs=$(echo $cfg | sed -n 's/.*CS=\([0-9]*\).*/\1/p'); sl=$(echo $cfg | sed -n 's/.*SLOTS=\([0-9]*\).*/\1/p')
  echo -n "$cfg: "; env ADAKV_DECODE_CS=$cs ${sl:+ADAKV_DECODE_SLOTS=$sl} timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])'
done; done
