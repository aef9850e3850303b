set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 300 python scripts/kbench.py --layers 4 > gpurun_out/kbench4.log 2>&1; echo "kbench exit $?"; tail -5 gpurun_out/kbench4.log
timeout 300 python scripts/kbench.py --layers 32 > gpurun_out/kbench32.log 2>&1; echo "kbench32 exit $?"; tail -5 gpurun_out/kbench32.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/kbench.py --layers 1 > gpurun_out/kbench1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_tc -s 4 -c 2 -o gpurun_out/prof_score_r1 python scripts/kbench.py --layers 1 > gpurun_out/ncu_score.log 2>&1; echo "ncu exit $?"; tail -5 gpurun_out/ncu_score.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r1.csv python scripts/kbench.py --layers 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu2 exit $?"
