import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2407_11550_b200 as A
from paper_2407_11550_b200.synthetic import planted_layer
L = A.lib(); dev = torch.device("cuda:0")
P, H, G, m, d, n = 1, 32, 8, 32, 128, 32768
q, k, v = planted_layer(P, H, G, n - m, m, d, seed=11, dtype=torch.bfloat16, device=dev)
cache = A.compress(q, k, v, 16384, reserve=64)
torch.cuda.synchronize()
print("budgets", cache.budgets.tolist())
dbg = torch.zeros(256 * 8, dtype=torch.int64, device=dev)
L.adakv_debug_set_decode_timestamps(C.c_void_p(dbg.data_ptr()))
qd = torch.randn((P, H, d), device=dev).to(torch.bfloat16)
kn = torch.randn((P, G, d), device=dev).to(torch.bfloat16); vn = torch.randn((P, G, d), device=dev).to(torch.bfloat16)
ws = torch.zeros(A.ops.decode_workspace_bytes(P, H, G, d, 4000), dtype=torch.uint8, device=dev)
for it in range(4):
    A.decode(qd, cache, kn, vn, max_rows=4000, ws=ws)
    torch.cuda.synchronize()
x = dbg.view(256, 8).cpu().numpy().astype(np.int64)
act = x[:, 0] > 0
t0 = x[act, 0].min()
for c, nm in enumerate(["start", "pre_wait", "post_wait", "computed", "partial_written", "group_done", "merge_done", "end"]):
    vals = x[act, c]; vals = vals[vals > 0]
    if len(vals): print(f"{nm:16s} min {(vals.min()-t0)/1e3:7.2f}  median {(np.median(vals)-t0)/1e3:7.2f}  max {(vals.max()-t0)/1e3:7.2f} us  (n={len(vals)})")
print("cluster size", A.lib().adakv_debug_decode_cluster(1, 8) if hasattr(A.lib(), "adakv_debug_decode_cluster") else "n/a")
