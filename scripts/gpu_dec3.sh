NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
ADAKV_DECODE_WARPS=16 NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
ADAKV_DECODE_WARPS=16 ADAKV_DECODE_CS=8 NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
ADAKV_DECODE_WARPS=16 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k decode 2>&1 | tail -2
