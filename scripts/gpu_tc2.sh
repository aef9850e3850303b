set -x
timeout 120 python scripts/tc_check.py > gpurun_out/tc_check.log 2>&1; echo "tc_check exit $?"; tail -12 gpurun_out/tc_check.log
timeout 200 python scripts/kbench.py --layers 4 > gpurun_out/kbench4.log 2>&1; echo "kbench exit $?"; tail -3 gpurun_out/kbench4.log
