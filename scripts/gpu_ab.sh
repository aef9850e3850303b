# A/B of builds of the library on one box: lib/ab_<V>.so for V in $VARIANTS (kbench, 32 layers)
L=paper_2407_11550_b200/lib
cp $L/libadakv_b200.so /tmp/cur.so
for r in 1 2; do for v in ${VARIANTS:-old new}; do cp $L/ab_$v.so $L/libadakv_b200.so; echo -n "$v: "; timeout 300 python scripts/kbench.py --layers 32 2>/dev/null | tail -1 | cut -c1-110; done; done
for v in ${VARIANTS:-old new}; do cp $L/ab_$v.so $L/libadakv_b200.so; echo -n "$v tests: "; timeout 600 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "score or compress or evict" 2>&1 | tail -1; done
cp /tmp/cur.so $L/libadakv_b200.so
