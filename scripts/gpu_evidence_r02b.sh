# Round-2 closing evidence: the bench line, then ncu captures (each after its plain run).
set -x
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
bash scripts/gpu_ncu.sh launches
bash scripts/gpu_ncu.sh traffic
bash scripts/gpu_ncu.sh decode
bash scripts/gpu_ncu.sh score
timeout 300 python scripts/kbench.py --layers 32 > gpurun_out/kbench_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -c 1 -o gpurun_out/prof_select32 \
    python scripts/kbench.py --layers 32 > gpurun_out/ncu_sel32.log 2>&1; echo "ncu select exit $?"
