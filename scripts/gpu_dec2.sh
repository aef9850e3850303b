for sl in 1 2 3; do
  echo "== slots $sl"
  ADAKV_DECODE_SLOTS=$sl timeout 300 python scripts/dec_ts2.py > gpurun_out/dec_ts2_$sl.log 2>&1; echo rc $?
  grep -E "graph:|cycles|p90|median" gpurun_out/dec_ts2_$sl.log; tail -6 gpurun_out/dec_ts2_$sl.log | head -2
done
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
