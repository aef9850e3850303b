timeout 100 python scripts/tc_time.py 1 > gpurun_out/tct.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 6 -c 2 -o gpurun_out/prof_score_v2b python scripts/tc_time.py 1 > gpurun_out/ncu_score.log 2>&1; echo "ncu $?"
