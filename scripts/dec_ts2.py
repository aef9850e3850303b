"""Per-launch decode timelines inside a CUDA graph (PDL chain over layers).

Each launch gets its own %globaltimer stamp buffer (ADAKV debug hook), so the overlap of
launch N+1's prologue with launch N is visible."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200 import pipeline as PL  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402

L = A.lib()
dev = torch.device("cuda:0")
Lyr, H, G, m, d, n = 4, 32, 8, 32, 128, 32768
qs, ks, vs = [], [], []
for l in range(Lyr):
    q, k, v = planted_layer(1, H, G, n - m, m, d, seed=11 + l, dtype=torch.bfloat16, device=dev)
    qs.append(q), ks.append(k), vs.append(v)
q = torch.stack(qs)
k = torch.stack(ks)
v = torch.stack(vs)
del qs, ks, vs
cache = PL.compress_model(q, k, v, 16384, reserve=64)
del q, k, v
torch.cuda.synchronize()
steps = int(os.environ.get("STEPS", "4"))
dg = PL.DecodeGraph(cache, Lyr, 1, 16384 + 64, use_graph=False)
nl = steps * Lyr
dbg = torch.zeros((nl, 256, 32), dtype=torch.int64, device=dev)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for s in range(steps):
            for l in range(Lyr):
                L.adakv_debug_set_decode_timestamps(None if os.environ.get('NOSTAMP') else C.c_void_p(dbg[s * Lyr + l].data_ptr()))
                seg = l * G
                A._lib.check(L.adakv_decode(
                    2, 1, H, G, d, 1, C.c_void_p(dg.q[l].data_ptr()), C.c_void_p(cache.k.data_ptr()),
                    C.c_void_p(cache.v.data_ptr()), cache.k.shape[0], C.c_void_p(cache.seg_start.data_ptr() + 4 * seg),
                    C.c_void_p(cache.seqlens.data_ptr() + 4 * seg), 16384 + 64, C.c_void_p(dg.k_new[l].data_ptr()),
                    C.c_void_p(dg.v_new[l].data_ptr()), C.c_void_p(dg.out[l].data_ptr()), C.c_void_p(dg.ws.data_ptr()),
                    dg.ws.numel(), C.c_void_p(st.cuda_stream)))
L.adakv_debug_set_decode_timestamps(None)
torch.cuda.synchronize()
for rep in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print("cluster", L.adakv_debug_decode_cluster(1, G))
print(f"graph: {nl} launches, {e0.elapsed_time(e1) * 1e3 / nl:.2f} us/launch")
if os.environ.get("NOSTAMP"):
    sys.exit(0)
x = dbg.cpu().numpy()
t0 = x[0][x[0][:, 0] > 0, 0].min()
names = ["start", "issued", "post_wait", "w0_done", "all_done", "pushed", "recvd", "end", "clwait", "q_in", "data0", "S0"]
order = [0, 1, 8, 2, 9, 10, 11, 3, 4, 5, 6, 7]
prev_end = None
for i in range(nl):
    a = x[i]
    act = a[:, 0] > 0
    row = []
    for c in order:
        vals = a[act, c]
        vals = vals[vals > 0]
        if len(vals) == 0:
            vals = np.array([t0])
        row.append(((vals.min() - t0) / 1e3, (vals.max() - t0) / 1e3))
    print(f"launch {i:2d} ctas {act.sum():3d} " + " ".join(f"{names[c]}[{lo:6.2f},{hi:6.2f}]" for c, (lo, hi) in zip(order, row)))

# intra-CTA durations from clock64 (cycles), median over CTAs of the last 8 launches
cyc = x[-8:, :, 16:]
act = cyc[:, :, 0] > 0
rel = cyc - cyc[:, :, :1]
print("clock64 cycles since CTA start (median over CTAs, last 8 launches):")
print("  med: " + "  ".join(f"{names[c]}={np.median(rel[:, :, c][act]):.0f}" for c in order if (cyc[:, :, c][act] > 0).any()))
print("  p90: " + "  ".join(f"{names[c]}={np.percentile(rel[:, :, c][act], 90):.0f}" for c in order if (cyc[:, :, c][act] > 0).any()))
gt = x[-1, :, :16]
print("globaltimer raw mod 1000 sample:", (gt[gt[:, 0] > 0][:4, :8] % 1000).tolist())
# per-cluster start times of one launch
cs = L.adakv_debug_decode_cluster(1, G)
a = x[-2]
act = a[:, 0] > 0
st0 = a[act, 0]
print("per-CTA start (us rel. to launch min), by cluster:")
for c in range(int(act.sum()) // cs):
    v = (a[c * cs:(c + 1) * cs, 0] - st0.min()) / 1e3
    print(f"  cluster {c}: " + " ".join(f"{t:5.2f}" for t in v))
pr = x[-8:, :, 12]
act = x[-8:, :, 0] > 0
vals = pr[act]
print("block0 landed at post_wait: ready", int((vals == 3).sum()), "not ready", int((vals == 2).sum()), "no blocks", int((vals < 2).sum()))
# per-warp loop-end times (globaltimer, us relative to the CTA's post_wait) and block counts
a = x[-3]
act = a[:, 0] > 0
print("per-warp loop end (us after this CTA's post_wait) / blocks, launch -3:")
for cta in np.nonzero(act)[0][:20]:
    pw = a[cta, 2]
    ends = [(a[cta, 24 + w] - pw) / 1e3 for w in range(8)]
    nbs = [int(a[cta, 8 + w]) for w in range(8)]
    print(f"  cta {cta:3d}: " + " ".join(f"{e:5.2f}/{n}" for e, n in zip(ends, nbs)) + f"   end {(a[cta, 7] - pw) / 1e3:5.2f}")
# warp-1 per-iteration clocks: [loop top, after mbar_wait, after LDS, after S] for blocks 0, 1
w1 = x[-8:, :, 8:16]
act = x[-8:, :, 0] > 0
v = w1[act]
v = v[(v[:, 0] > 0) & (v[:, 4] > 0)]
rel = v - v[:, :1]
print("warp1 cycles (median): blk0 wait", int(np.median(rel[:, 1])), "lds", int(np.median(rel[:, 2] - rel[:, 1])),
      "S", int(np.median(rel[:, 3] - rel[:, 2])), "| blk0 S->blk1 top", int(np.median(rel[:, 4] - rel[:, 3])),
      "blk1 wait", int(np.median(rel[:, 5] - rel[:, 4])), "lds", int(np.median(rel[:, 6] - rel[:, 5])), "S", int(np.median(rel[:, 7] - rel[:, 6])))
