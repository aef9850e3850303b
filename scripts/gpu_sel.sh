timeout 300 python scripts/sel_ts.py 2>&1 | tail -2
timeout 300 python scripts/kbench.py --layers 32 2>&1 | tail -1 | cut -c1-250
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
