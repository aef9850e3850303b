NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|rror"
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
