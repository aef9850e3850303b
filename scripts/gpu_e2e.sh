timeout 600 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "compress" 2>&1 | tail -2
for r in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench_e2e.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"], d["compress_ms_per_layer"], d["e2e"])'; done
