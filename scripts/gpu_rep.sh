for b in 2048 3072 4096; do echo "== P8 BUD $b"; P=8 BUD=$b timeout 120 python scripts/dec_repro.py 2>&1 | grep -E "cluster|ok|Error" | head -2; done
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
