timeout 120 python scripts/dec_ts.py
timeout 200 python scripts/kbench.py --layers 4 | tail -1
