set -x
timeout 300 python scripts/kbench.py --layers 1 > gpurun_out/kbench1.log 2>&1; echo "kbench1 exit $?"; tail -2 gpurun_out/kbench1.log
timeout 300 python scripts/kbench.py --layers 4 > gpurun_out/kbench4.log 2>&1; echo "kbench4 exit $?"; tail -2 gpurun_out/kbench4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 2 -c 1 -o gpurun_out/prof_select_r1 python scripts/kbench.py --layers 1 > gpurun_out/ncu_sel.log 2>&1; echo "ncu sel $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 5 -c 1 -o gpurun_out/prof_decode_r1 python scripts/kbench.py --layers 1 > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 4 -c 2 -o gpurun_out/prof_score_r1b python scripts/kbench.py --layers 1 > gpurun_out/ncu_score2.log 2>&1; echo "ncu score $?"
