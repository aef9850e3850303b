set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python scripts/kbench.py --layers 4 > gpurun_out/kbench.log 2>&1; echo "kbench exit $?"; tail -8 gpurun_out/kbench.log
timeout 600 python bench.py --layers 2 --decode-steps 16 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo "bench exit $?"; tail -3 gpurun_out/bench_small.log
