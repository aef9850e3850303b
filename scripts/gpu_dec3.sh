for cs in 6 8 9 10 11 12 14 16; do
export ADAKV_DECODE_CS=$cs
echo "cs $cs $(NOSTAMP=1 STEPS=32 timeout 120 python scripts/dec_ts2.py 2>&1 | grep -E 'graph')"
done
