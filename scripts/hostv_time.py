"""Compress of config 2 (32 layers, 32K prompt) with V in device memory vs pinned host memory
(the gather reads the retained + window rows over the host link), alone and while a large
H2D copy runs on another stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_11550_b200 import pipeline as PL  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402

dev = torch.device("cuda:0")
Lyr, H, G, m, d, n = 32, 32, 8, 32, 128, 32768
LB = 2048 * G
q, k, v = planted_layer(Lyr, H, G, n - m, m, d, seed=1, dtype=torch.bfloat16, device=dev)
q, k, v = q.reshape(Lyr, 1, H, m, d), k.reshape(Lyr, 1, G, n, d), v.reshape(Lyr, 1, G, n, d)
vh = v.cpu().pin_memory()
cache = PL.compress_model(q, k, v, LB, reserve=8)
big_h = torch.empty(2 * 1024**3, dtype=torch.uint8).pin_memory()
big_d = torch.empty_like(big_h, device=dev)
cst = torch.cuda.Stream()


def timed(vv, copy=False, reps=5):
    for _ in range(2):
        PL.compress_model(q, k, vv, LB, reserve=8, out=cache)
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(cst):
            big_d.copy_(big_h, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        PL.compress_model(q, k, vv, LB, reserve=8, out=cache)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for r in range(2):
    print(f"device V: {timed(v):.2f} ms  host V: {timed(vh):.2f} ms  host V + concurrent H2D: {timed(vh, True):.2f} ms"
          f"  device V + concurrent H2D: {timed(v, True):.2f} ms")

# decode (one graph = one step over 32 layers, replayed 256 times) alone vs under a 2 GB H2D
dcache = PL.compress_model(q, k, v, LB, reserve=300)
dg = PL.DecodeGraph(dcache, Lyr, 1, LB + 300)
seq0 = dcache.seqlens.clone()


def dec(copy=False, steps=256):
    dcache.seqlens.copy_(seq0)
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(cst):
            big_d.copy_(big_h, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dg.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (steps * Lyr)


dec()
for r in range(2):
    print(f"decode us/step-layer: alone {dec():.3f}  under H2D {dec(True):.3f}")
