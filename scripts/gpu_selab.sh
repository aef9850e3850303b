# Select-kernel change check: parity tests touching select/compress, then latency.
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/sel_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/sel_pytest.log
timeout 300 python scripts/select_bench.py > gpurun_out/sel_bench.log 2>&1; tail -c 400 gpurun_out/sel_bench.log
timeout 300 python scripts/kbench.py --layers 32 > gpurun_out/sel_kbench.log 2>&1; tail -1 gpurun_out/sel_kbench.log
