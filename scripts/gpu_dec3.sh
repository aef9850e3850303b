for cs in auto 8; do for sl in 2 3; do
echo "== cs $cs slots $sl"
if [ $cs = auto ]; then unset ADAKV_DECODE_CS; else export ADAKV_DECODE_CS=$cs; fi
ADAKV_DECODE_SLOTS=$sl NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E "graph|cluster|rror"
done; done
unset ADAKV_DECODE_CS
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
