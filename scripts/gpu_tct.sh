for dbg in 1 513 65; do ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_time.py 8 2>&1 | tail -1; done
