for cs in auto 10 11; do
echo "== W8 cs $cs"; if [ $cs = auto ]; then unset ADAKV_DECODE_CS; else export ADAKV_DECODE_CS=$cs; fi
NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
done
cp paper_2407_11550_b200/lib_w12/libadakv_b200.so paper_2407_11550_b200/lib/libadakv_b200.so
for cs in auto 10 11 12; do
echo "== W12 cs $cs"; if [ $cs = auto ]; then unset ADAKV_DECODE_CS; else export ADAKV_DECODE_CS=$cs; fi
NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
done
unset ADAKV_DECODE_CS
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k decode 2>&1 | tail -2
