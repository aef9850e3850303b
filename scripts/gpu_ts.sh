for m in 0 3; do echo "== qmode $m"; ADAKV_DECODE_QMODE=$m timeout 300 python scripts/dec_ts4.py 2>&1 | grep -v "^ *[0-9]* n" | tail -30; done
