python - <<'PY'
import paper_2407_11550_b200 as A
L = A.lib()
print("cluster", L.adakv_debug_decode_cluster(1, 8))
PY
timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])'
