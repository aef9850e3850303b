# K1 slice-size A/B and the pass-2 L2 evidence (one gpurun call):
#   per ADAKV_SCORE_SLICE_MB: scoring time per layer over 32 layers (scripts/kbench.py);
#   then ncu with --cache-control none (L2 left as the previous kernel left it, one replay pass
#   per kernel) over 4 slices' (pass 1, pass 2) pairs: dram bytes read per pass.
for mb in 24 48 64 96; do
  echo "slice ${mb} MB: $(ADAKV_SCORE_SLICE_MB=$mb timeout 300 python scripts/kbench.py --layers 32 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["score_ms_per_layer"], d["compress_ms_per_layer"])')"
done
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
  -k regex:score_tc -s 8 -c 8 python scripts/kbench.py --layers 8 > gpurun_out/ncu_l2.log 2>&1
grep -E "score_tc_kernel|dram__bytes_read|lts__t_sector_hit|gpu__time" gpurun_out/ncu_l2.log | head -40
