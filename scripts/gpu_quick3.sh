timeout 800 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python scripts/select_bench.py 2>&1 | tail -1 | cut -c1-300
P=1 timeout 300 python scripts/sel_ts.py 2>&1 | tail -2
