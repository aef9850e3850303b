"""Per-phase clock64 stamps of the select kernel on one config-2 layer (debug hook)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402

L = A.lib()
dev = torch.device("cuda:0")
P = int(os.environ.get("P", "1"))
H, G, m, d, n = 32, 8, 32, 128, int(os.environ.get("PROMPT", "32768"))
q, k, v = planted_layer(P, H, G, n - m, m, d, seed=3, dtype=torch.bfloat16, device=dev)
A.compress(q, k, v, 16384, reserve=64)
torch.cuda.synchronize()
dbg = torch.zeros((P * 16, 32), dtype=torch.int64, device=dev)
L.adakv_debug_set_select_timestamps(C.c_void_p(dbg.data_ptr()))
for _ in range(3):
    A.compress(q, k, v, 16384, reserve=64)
torch.cuda.synchronize()
L.adakv_debug_set_select_timestamps(None)
x = dbg.cpu().numpy()
act = x[:, 0] > 0
rel = x[act] - x[act][:, :1]
n_st = int((x[act][:, :24] > 0).sum(axis=1).max())
print("CTAs", int(act.sum()), "stamps", n_st)
print("median cycles since start:", [int(np.median(rel[:, i])) for i in range(n_st)])
print("max    cycles since start:", [int(np.max(rel[:, i])) for i in range(n_st)])
fine = x[act][:, 24:31]
if (fine > 0).all():
    d = np.diff(fine, axis=1)
    print("radix pass 1 phases (key loop, sync, warp-sum+sync, cluster.sync, DSMEM sum, sync):",
          [int(np.median(d[:, i])) for i in range(d.shape[1])])
