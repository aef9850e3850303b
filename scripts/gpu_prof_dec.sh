timeout 300 python scripts/kbench.py --layers 1 > gpurun_out/kbench1.log 2>&1 && \
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:decode_tc -s 5 -c 3 -o gpurun_out/prof_decode_v6 python scripts/kbench.py --layers 1 > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec $?"; tail -3 gpurun_out/ncu_dec.log
