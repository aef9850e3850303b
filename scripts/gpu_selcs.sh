for cs in 8 4 3 2; do echo -n "CS=$cs: "; ADAKV_SELECT_CS=$cs timeout 300 python scripts/kbench.py --layers 32 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["select_us_per_call"], d["compress_ms_per_layer"])'; done
for cs in 4; do ADAKV_SELECT_CS=$cs timeout 600 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "select or compress" 2>&1 | tail -1; done
ADAKV_SELECT_CS=4 timeout 300 python scripts/select_bench.py 2>&1 | tail -6
timeout 300 python scripts/select_bench.py 2>&1 | tail -6
