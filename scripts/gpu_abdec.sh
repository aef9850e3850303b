# decode A/B of lib/ab_old.so vs lib/ab_new.so: parity tests on new, bench decode timing interleaved
L=paper_2407_11550_b200/lib
cp $L/libadakv_b200.so /tmp/cur.so
cp $L/ab_new.so $L/libadakv_b200.so
timeout 600 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "decode or smoke" 2>&1 | tail -3
for r in 1 2; do for v in old new; do cp $L/ab_$v.so $L/libadakv_b200.so; echo -n "$v: "; timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])'; done; done
cp /tmp/cur.so $L/libadakv_b200.so
