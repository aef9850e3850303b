"""UMMA decode per-CTA phase timeline (globaltimer) inside the PDL graph chain (4 layers)."""
import ctypes as C
import os
import sys
os.environ.setdefault("ADAKV_DECODE_UMMA", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200 import pipeline as PL  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402

L = A.lib()
dev = torch.device("cuda:0")
Lyr, H, G, m, d, n = 8, 32, 8, 32, 128, 32768
q, k, v = planted_layer(Lyr, H, G, n - m, m, d, seed=11, dtype=torch.bfloat16, device=dev)
cache = PL.compress_model(q.view(Lyr, 1, H, m, d), k.view(Lyr, 1, G, n, d), v.view(Lyr, 1, G, n, d), 16384, reserve=64)
del q, k, v
torch.cuda.synchronize()
dg = PL.DecodeGraph(cache, Lyr, 1, 16384 + 64, use_graph=False)
steps = 3
nl = steps * Lyr
dbg = torch.zeros((nl, 256, 32), dtype=torch.int64, device=dev)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for s in range(steps):
            for l in range(Lyr):
                L.adakv_debug_set_decode_timestamps(C.c_void_p(dbg[s * Lyr + l].data_ptr()))
                seg = l * G
                A._lib.check(L.adakv_decode(
                    2, 1, H, G, d, 1, C.c_void_p(dg.q[l].data_ptr()), C.c_void_p(cache.k.data_ptr()),
                    C.c_void_p(cache.v.data_ptr()), cache.k.shape[0], C.c_void_p(cache.seg_start.data_ptr() + 4 * seg),
                    C.c_void_p(cache.seqlens.data_ptr() + 4 * seg), 16384 + 64, C.c_void_p(dg.k_new[l].data_ptr()),
                    C.c_void_p(dg.v_new[l].data_ptr()), C.c_void_p(dg.out[l].data_ptr()), C.c_void_p(dg.ws.data_ptr()),
                    dg.ws.numel(), C.c_void_p(st.cuda_stream)))
L.adakv_debug_set_decode_timestamps(None)
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
x = dbg.cpu().numpy()
names = ["start", "post_wait", "q_ready", "s_done", "smax", "pv_issued", "o_done", "pushed", "recvd", "end"]
for i in range(nl - 4, nl):
    a = x[i]
    act = a[:, 0] > 0
    t0 = x[i - 1][x[i - 1][:, 0] > 0, 9].max()  # previous launch end
    print(f"launch {i}: " + " ".join(f"{nm}[{(a[act, c].min() - t0) / 1e3:5.2f},{(a[act, c].max() - t0) / 1e3:5.2f}]"
                                      for c, nm in enumerate(names)))
