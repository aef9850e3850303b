for b in 1 2 4 8; do echo "batch $b: $(BATCH=$b NOSTAMP=1 timeout 300 python scripts/dec_ts4.py 2>&1 | tail -1)"; done
