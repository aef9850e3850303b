for dbg in 0 0 1024; do ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_time.py 8 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
cp paper_2407_11550_b200/lib/libadakv_b200.so /tmp/new.so
cp paper_2407_11550_b200/lib/prof_libadakv.so paper_2407_11550_b200/lib/libadakv_b200.so
for dbg in 0; do echo "== $dbg"; ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_ts2.py 2>&1 | tail -14; done
cp /tmp/new.so paper_2407_11550_b200/lib/libadakv_b200.so
