set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -20 gpurun_out/smoke.log
timeout 600 python bench.py --layers 2 --decode-steps 16 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo "bench exit $?"; tail -20 gpurun_out/bench_small.log
