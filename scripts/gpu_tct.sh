for dbg in 0 1024 1; do ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_time.py 8 2>&1 | tail -1; done
