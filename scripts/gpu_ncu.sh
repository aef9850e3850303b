# One ncu pass per gpurun call (after the same command has exited 0 without ncu):
#   bash scripts/gpu_ncu.sh launches|decode|score|select|gather|traffic
CMD="python bench.py --layers 2 --decode-steps 16 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
case "$1" in
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ;;
  decode) timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 40 -c 2 -o gpurun_out/prof_decode $CMD > gpurun_out/ncu_dec.log 2>&1 ;;
  score) timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_tc -s 2 -c 2 -o gpurun_out/prof_score $CMD > gpurun_out/ncu_score.log 2>&1 ;;
  select) timeout 900 ncu --set full --clock-control none --import-source on -k regex:select -s 1 -c 1 -o gpurun_out/prof_select $CMD > gpurun_out/ncu_sel.log 2>&1 ;;
  traffic) timeout 600 python scripts/decode_traffic.py > gpurun_out/traffic_plain.json 2>&1 && \
    timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:decode_tc -s 8193 -c 1 --csv python scripts/decode_traffic.py > gpurun_out/ncu_traffic.csv 2>&1 ;;
  gather) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel|layout_kernel" -s 2 -c 2 -o gpurun_out/prof_gather $CMD > gpurun_out/ncu_gather.log 2>&1 ;;
esac
echo "ncu $1 exit $?"
