set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python scripts/kbench.py --layers 4 > gpurun_out/kbench4.log 2>&1; echo "kbench exit $?"; tail -3 gpurun_out/kbench4.log
