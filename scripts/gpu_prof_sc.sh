timeout 120 python scripts/tc_time.py 2 > gpurun_out/tct.log 2>&1 && \
timeout 600 ncu --set full --warp-sampling-interval 2 --clock-control none --import-source on -k regex:score_tc_kernel -s 6 -c 2 -o gpurun_out/prof_score_p12 python scripts/tc_time.py 2 > gpurun_out/ncu_sc.log 2>&1; echo "ncu $?"; tail -2 gpurun_out/ncu_sc.log
