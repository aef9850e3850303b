for dbg in 0; do ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_time.py 8 2>&1 | tail -1; ADAKV_TC_DEBUG=$dbg timeout 120 python scripts/tc_time.py 8 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
