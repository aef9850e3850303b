"""Segment-length spread of the bench's compressed caches (config 2): per layer min / max /
max-over-mean of the 8 KV-group segments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2407_11550_b200 import pipeline as PL
from paper_2407_11550_b200.synthetic import planted_layer
dev = torch.device("cuda:0")
L, B, H, G, d, m, n = 32, 1, 32, 8, 128, 32, 32768
q, k, v = planted_layer(L * B, H, G, n - m, m, d, seed=1000, dtype=torch.bfloat16, device=dev)
cache = PL.compress_model(q.reshape(L, B, H, m, d), k.reshape(L, B, G, n, d), v.reshape(L, B, G, n, d), 2048 * G, reserve=8)
s = cache.seqlens.cpu().numpy().reshape(L, G)
r = s.max(1) / s.mean(1)
print("per-layer max/mean:", np.round(r, 2).tolist())
print("overall: min seg", s.min(), "max seg", s.max(), "mean", s.mean(), "median max/mean", np.median(r))
