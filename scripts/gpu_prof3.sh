timeout 200 python scripts/kbench.py --layers 1 > gpurun_out/kbench1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 4 -c 2 -o gpurun_out/prof_score_v2 python scripts/kbench.py --layers 1 > gpurun_out/ncu_score.log 2>&1; echo "ncu $?"
