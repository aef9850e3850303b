for dbg in 0 1 0 1; do ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_time.py 8 2>&1 | tail -1; done
timeout 800 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
