timeout 300 python scripts/dec_ts4.py 2>&1 | grep -v Warn | grep "clk\|warp loop\|graph\|next first\|warp1"
NOSTAMP=1 timeout 300 python scripts/dec_ts4.py 2>&1 | tail -1
