timeout 800 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 300 python scripts/kbench.py --layers 32 2>&1 | tail -3 | head -2 | cut -c1-200; done
