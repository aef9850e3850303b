# K1 exp2 split sweep (how many of every 8 exp2 run as an FMA-pipe polynomial) per pass:
# rebuilds score_window_tc.cu with EXTRA flags and times scoring over 32 layers (kbench).
for p1 in 0 2 4; do for p2 in 0 2; do
  touch paper_2407_11550_b200/csrc/score_window_tc.cu
  make -s -j8 -C paper_2407_11550_b200/csrc EXTRA="-DADAKV_PASS1_POLY=$p1 -DADAKV_PASS2_POLY=$p2" 2>&1 | grep -v spill | grep -v "^$"
  echo "pass1 $p1 pass2 $p2: $(timeout 300 python scripts/kbench.py --layers 32 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["score_ms_per_layer"])')"
done; done
touch paper_2407_11550_b200/csrc/score_window_tc.cu; make -s -j8 -C paper_2407_11550_b200/csrc 2>&1 | grep -v spill | grep -v "^$"
