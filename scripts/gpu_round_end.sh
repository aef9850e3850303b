# Round-end evidence in one gpurun call: final run (tests, smoke, bench, reference arm,
# per-stage timings), then the ncu captures (decode, score) and the launch list.
bash scripts/gpu_final.sh
bash scripts/gpu_ncu.sh decode
bash scripts/gpu_ncu.sh score
bash scripts/gpu_ncu.sh launches
