import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADAKV_TC_DEBUG"] = sys.argv[1] if len(sys.argv) > 1 else "33"
import torch, numpy as np
import paper_2407_11550_b200 as A
from paper_2407_11550_b200.synthetic import planted_layer
L = A.lib(); dev = torch.device("cuda:0")
q, k, v = planted_layer(1, 32, 8, 32736, 32, 128, seed=11, dtype=torch.bfloat16, device=dev)
gs = torch.empty((1, 8, 32736), dtype=torch.float32, device=dev)
dbg = torch.zeros(148 * 8, dtype=torch.int64, device=dev)
shape = A.ops.layer_shape(1, 32, 8, 32, 32736, 128)
nb = C.c_size_t(); A._lib.check(L.adakv_window_scores_workspace(2, C.byref(shape), C.byref(nb)))
ws = torch.zeros(nb.value * 2, dtype=torch.uint8, device=dev)
for it in range(3):
    dbg.zero_()
    A._lib.check(L.adakv_window_scores(2, C.byref(shape), 7, 1, C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(dbg.data_ptr()),
        C.c_void_p(gs.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
d = dbg.view(148, 8).cpu().numpy().astype(float)
act = d[:, 6] > 0
print("debug", os.environ["ADAKV_TC_DEBUG"], "CTAs", act.sum(), "tiles/CTA", d[act, 6].mean())
names = ["prod_wait_empty", "prod_total", "mma_wait_acc_empty", "mma_wait_full", "epi_wait_acc_full", "epi_total"]
for i, nm in enumerate(names):
    print(f"{nm:22s} mean {d[act, i].mean():10.0f}  max {d[act, i].max():10.0f} cycles")
