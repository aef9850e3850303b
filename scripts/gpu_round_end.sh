# Round-end evidence in one gpurun call: final run (tests, smoke, bench, reference arm,
# per-stage timings), then the decode ncu capture and the launch list.
bash scripts/gpu_final.sh
bash scripts/gpu_ncu.sh decode
bash scripts/gpu_ncu.sh launches
