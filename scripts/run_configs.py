"""Run the supplementary BASELINE-config fields of bench.py alone (one GPU):
    python scripts/run_configs.py [config3 config4 config5]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import bench_configs as B  # noqa: E402

dev = torch.device("cuda:0")
peak = 6531.0
for name in sys.argv[1:] or ["config3", "config4", "config5"]:
    print(name, json.dumps(getattr(B, name)(dev, peak, 0, 1)), flush=True)
