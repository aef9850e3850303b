cp paper_2407_11550_b200/lib/libadakv_b200.so /tmp/lib_new.so
for r in 1 2; do
cp /tmp/lib_new.so paper_2407_11550_b200/lib/libadakv_b200.so
echo "new $(timeout 900 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])')"
cp paper_2407_11550_b200/lib_prev/libadakv_b200.so paper_2407_11550_b200/lib/libadakv_b200.so
echo "prev $(timeout 900 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"])')"
done
