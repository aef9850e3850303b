"""Role wait counters of the two scoring passes (clock64 cycles, per CTA) at the config-2 layer shape."""
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
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1
q, k, v = planted_layer(P, 32, 8, 32736, 32, 128, seed=11, dtype=torch.bfloat16, device=dev)
dbg = torch.zeros(2 * 160 * 16, dtype=torch.int64, device=dev)
for it in range(3):
    if it == 2:
        L.adakv_debug_set_score_counters(C.c_void_p(dbg.data_ptr()))
    A.window_scores(q, k, 7)
    torch.cuda.synchronize()
L.adakv_debug_set_score_counters(None)
d = dbg.view(2, 160, 16).cpu().numpy().astype(float)
names = {0: "prod_wait_empty", 1: "prod_total", 2: "mma_wait_acc_empty", 3: "mma_wait_full", 7: "mma_wait_e_full",
         8: "mma_wait_d2_empty", 4: "epi_wait_acc_full", 5: "epi_total", 6: "tiles"}
for ps in range(2):
    act = d[ps, :, 6] > 0
    print(f"pass {ps + 1}: CTAs {int(act.sum())}")
    for i, nm in names.items():
        print(f"   {nm:20s} mean {d[ps, act, i].mean():10.0f}  max {d[ps, act, i].max():10.0f}")
