python -c "
import paper_2407_11550_b200 as A
L = A.lib()
print('cluster segs 8:', L.adakv_debug_decode_cluster(1, 8), ' segs 16:', L.adakv_debug_decode_cluster(2, 8), ' segs 2:', L.adakv_debug_decode_cluster(1, 2))"
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])'; done
timeout 800 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
