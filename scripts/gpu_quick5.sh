timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bq.log 2>&1; echo "exit $?"; tail -2 gpurun_out/bq.log | cut -c1-200
tail -1 gpurun_out/bq.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["decode_us_per_layer_step"], d.get("decode_batch_scaling"))'
