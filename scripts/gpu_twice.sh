L=paper_2407_11550_b200/lib
cp $L/libadakv_b200.so /tmp/cur.so
for v in T1 T2 T3; do cp $L/ab_$v.so $L/libadakv_b200.so; echo "== $v"; timeout 300 python scripts/dec_ts4.py 2>&1 | grep -E "cluster|post_wait -> loop0|clk post_wait|warp1"; done
cp /tmp/cur.so $L/libadakv_b200.so
