"""Quick TC-vs-generic-vs-oracle check of window scoring (run under `timeout`)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_11550_b200 as A
from paper_2407_11550_b200.synthetic import planted_layer
from oracle import oracle as O

L = A.lib()
dev = torch.device("cuda:0")
for (P, H, G, n_o, pk) in [(1, 4, 1, 1000, 7), (1, 32, 8, 4064, 7), (2, 8, 4, 777, 5), (1, 4, 2, 300, 3), (1, 8, 2, 129, 1)]:
    q, k, v = planted_layer(P, H, G, n_o, 32, 128, seed=3, dtype=torch.bfloat16, device=dev)
    L.adakv_set_tensor_core_scoring(1)
    t0 = time.time()
    gs_tc, hs_tc = A.window_scores(q, k, pk, head_scores=True)
    torch.cuda.synchronize()
    t1 = time.time()
    L.adakv_set_tensor_core_scoring(0)
    gs_g, hs_g = A.window_scores(q, k, pk, head_scores=True)
    torch.cuda.synchronize()
    d = (gs_tc - gs_g).abs().max().item()
    mx = gs_g.abs().max().item()
    dh = (hs_tc - hs_g).abs().max().item()
    q64 = q.double().cpu().numpy(); k64 = k.double().cpu().numpy()
    gsz = H // G
    per = [O.window_scores(q64[0, h], k64[0, 0, :n_o], pk) for h in range(gsz)]
    ref = O.group_mean_scores(np.stack(per), gsz)[0]
    e_tc = np.abs(gs_tc[0, 0].double().cpu().numpy() - ref).max()
    e_g = np.abs(gs_g[0, 0].double().cpu().numpy() - ref).max()
    print(f"P={P} H={H} G={G} n_o={n_o} k={pk}: |tc-generic|={d:.3e} (max {mx:.3e}) heads {dh:.3e}; vs oracle tc={e_tc:.3e} generic={e_g:.3e} rel={e_tc/ref.max():.2e} t={1e3*(t1-t0):.1f}ms", flush=True)
L.adakv_set_tensor_core_scoring(1)
# timing at the config-2 layer shape
q, k, v = planted_layer(1, 32, 8, 32736, 32, 128, seed=5, dtype=torch.bfloat16, device=dev)
for it in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); A.window_scores(q, k, 7); e1.record(); torch.cuda.synchronize()
    print("32K layer scoring ms", e0.elapsed_time(e1))
