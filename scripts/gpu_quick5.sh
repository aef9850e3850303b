for cs in 5 6 7 8 9; do echo "B2 cs $cs: $(BATCH=2 ADAKV_DECODE_CS=$cs NOSTAMP=1 timeout 300 python scripts/dec_ts4.py 2>&1 | tail -1)"; done
for cs in 3 4 5; do echo "B4 cs $cs: $(BATCH=4 ADAKV_DECODE_CS=$cs NOSTAMP=1 timeout 300 python scripts/dec_ts4.py 2>&1 | tail -1)"; done
