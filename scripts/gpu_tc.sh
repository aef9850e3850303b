set -x
timeout 120 python scripts/tc_check.py > gpurun_out/tc_check.log 2>&1; echo "tc_check exit $?"; cat gpurun_out/tc_check.log | tail -30
