"""Per-launch decode timelines at the bench's decode shape (32 layers x 8 groups, ~2048 rows
per group with adaptive spread; the caches exceed L2), PDL chain inside a CUDA graph."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200 import pipeline as PL  # noqa: E402
from paper_2407_11550_b200.ops import CompressedCache  # noqa: E402

L = A.lib()
if os.environ.get("NOPDL"):
    L.adakv_set_decode_overlap(0)
dev = torch.device("cuda:0")
Lyr, H, G, d = int(os.environ.get("LAYERS", "32")), 32, 8, 128
LB = int(os.environ.get("LBH", "2048")) * G
B = int(os.environ.get("BATCH", "1"))
steps = int(os.environ.get("STEPS", "4"))
reserve = steps + 8
rng = np.random.default_rng(0)
lens = []
for l in range(Lyr * B):
    w = rng.lognormal(0, float(os.environ.get("SKEW", "0.05")), G)
    x = np.floor(w / w.sum() * LB).astype(np.int64)
    x[0] += LB - x.sum()
    lens.append(x)
lens = np.concatenate(lens).astype(np.int32)
caps = lens + reserve
starts = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int32)
rows = int(caps.sum())
kp = (torch.randn((rows, d), device=dev) * 0.5).to(torch.bfloat16)
vp = torch.randn((rows, d), device=dev).to(torch.bfloat16)
cache = CompressedCache(k=kp, v=vp, seg_start=torch.as_tensor(starts, device=dev), seqlens=torch.as_tensor(lens, device=dev),
                        budgets=torch.as_tensor(lens, device=dev), P=Lyr * B, H=H, G=G, m=0, d=d, reserve=reserve,
                        layer_budget=LB)
dg = PL.DecodeGraph(cache, Lyr, B, int(caps.max()), use_graph=False)
dg.q.normal_()
nl = steps * Lyr
dbg = torch.zeros((nl, 256, 64), dtype=torch.int64, device=dev)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
stamp = not os.environ.get("NOSTAMP")
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for s in range(steps):
            for l in range(Lyr):
                L.adakv_debug_set_decode_timestamps(C.c_void_p(dbg[s * Lyr + l].data_ptr()) if stamp else None)
                PL.decode_layer(L, cache, l, B, dg.q[l], dg.k_new[l], dg.v_new[l], dg.out[l], dg.ws, int(caps.max()),
                                C.c_void_p(st.cuda_stream), chained=s > 0 or l > 0)
L.adakv_debug_set_decode_timestamps(None)
torch.cuda.synchronize()
seq0 = cache.seqlens.clone()
g.replay()
cache.seqlens.copy_(seq0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
tm = False
cs = L.adakv_debug_decode_cluster(B, G)
print(f"kernel tc cluster {cs}; graph: {nl} launches, {e0.elapsed_time(e1) * 1e3 / nl:.2f} us/launch; segment rows {lens.min()}..{lens.max()}")
if not stamp:
    sys.exit(0)
x = dbg.cpu().numpy()
names = (["start", "issued", "post_wait", "p_done", "o_done", "pushed", "recvd", "end"] if tm else
         ["start", "issued", "post_wait", "loop0", "merged", "pushed", "recvd", "end"])
base = x[nl // 2][x[nl // 2][:, 0] > 0, 0].min()
print("launch: [min,max] per stamp, us relative to launch", nl // 2, "first start")
for i in range(nl // 2, min(nl, nl // 2 + 12)):
    a = x[i]
    act = a[:, 0] > 0
    cols = []
    for c in range(8):
        v = a[act, c]
        cols.append(f"{names[c]}[{(v.min() - base) / 1e3:6.2f},{(v.max() - base) / 1e3:6.2f}]")
    print(f"{i:3d} n{act.sum():3d} " + " ".join(cols))
# per-CTA phase durations (globaltimer ns), medians over the second half of the launches
half = x[nl // 2:]
act = half[:, :, 0] > 0
def med(a, b):
    return np.median((half[:, :, b] - half[:, :, a])[act]) / 1e3
def p90(a, b):
    return np.percentile((half[:, :, b] - half[:, :, a])[act], 90) / 1e3
for a_, b_ in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (0, 7), (2, 7)]:
    print(f"  {names[a_]:>9s} -> {names[b_]:<9s} med {med(a_, b_):5.2f} p90 {p90(a_, b_):5.2f} us")
# launch-level: first start of i+1 vs last end of i; post_wait(i+1) vs end(i)
gaps, rel, span = [], [], []
for i in range(nl // 2, nl - 1):
    a, b = x[i], x[i + 1]
    ea = a[a[:, 0] > 0, 7].max()
    sb = b[b[:, 0] > 0, 0]
    pb = b[b[:, 0] > 0, 2]
    gaps.append((sb.min() - ea) / 1e3)
    rel.append((pb.min() - ea) / 1e3)
    span.append((ea - a[a[:, 0] > 0, 0].min()) / 1e3)
print(f"next first start - this last end: med {np.median(gaps):.2f} us; next first post_wait - this last end: med {np.median(rel):.2f}; launch span med {np.median(span):.2f}")
# warp loop ends relative to post_wait
lw = (half[:, :, 24:32] - half[:, :, 2:3])[act] / 1e3
print("warp loop end after post_wait: med", np.round(np.median(lw, axis=0), 2), "max", np.round(lw.max(axis=0), 2))
# clock64 (cycles) per-CTA phase durations: slots 16 + k
ck = half[:, :, 16:24]
for a_, b_ in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7)]:
    dd = (ck[:, :, b_] - ck[:, :, a_])[act]
    print(f"  clk {names[a_]:>9s} -> {names[b_]:<9s} med {np.median(dd):7.0f} p90 {np.percentile(dd, 90):7.0f} cycles")
# consistency: merged (globaltimer) vs max warp loop end
me = half[:, :, 4][act]
wl = half[:, :, 24:32][act].max(axis=1)
print("merged - max warp loop end (us): med", np.median((me - wl) / 1e3), "min", ((me - wl) / 1e3).min())
if tm:
    ck8 = half[:, :, 8:12][act]
    pw = half[:, :, 18][act]
    r = ck8 - pw[:, None]
    print("ds warp-0 cycles after post_wait: pre-Q-wait %d, Q landed %d, S max done %d, P stored %d" %
          tuple(np.median(r, axis=0)))
    st0 = half[:, :, 16][act]
    print("ds prologue (cycles after start): loads %d, inits %d, TMA issued %d" % (
        np.median(half[:, :, 13][act] - st0), np.median(half[:, :, 14][act] - st0), np.median(half[:, :, 12][act] - st0)))
    landed = half[:, :, 15][act] - half[:, :, 18][act]
    print("ds all blocks landed, cycles relative to post_wait: med %d p10 %d p90 %d" % (
        np.median(landed), np.percentile(landed, 10), np.percentile(landed, 90)))
    print("  p90: %d %d %d %d" % tuple(np.percentile(r, 90, axis=0)))
    sys.exit(0)
# warp 1's first two blocks (cycles): slots 8..15 = [top, data, S, end] x 2; relative to post_wait clock
w1 = half[:, :, 8:16][act]
pw = ck[:, :, 2][act]
ok = w1[:, 4] > 0
if ok.sum() == 0:
    sys.exit(0)
r = (w1[ok] - pw[ok][:, None])
print("warp1 (CTAs with >=2 blocks):", ok.sum(), "med cycles after post_wait: top0 %d data0 %d S0 %d end0 %d top1 %d data1 %d Qlanded %d end1 %d" % tuple(np.median(r, axis=0)))
print("  p90: top0 %d data0 %d S0 %d end0 %d top1 %d data1 %d Qlanded %d end1 %d" % tuple(np.percentile(r, 90, axis=0)))
pw4 = half[:, :, 18][act]
ww = half[:, :, 32:64][act].reshape(-1, 8, 4)
okw = ww[:, :, 1] > 0
print("per-warp cycles after post_wait (median over CTAs/launches): Q landed | first pair S done | first pair PV done | loop end")
for w in range(8):
    sel = okw[:, w]
    r = ww[sel, w, :] - pw4[sel][:, None]
    print(f"  warp {w}: " + " ".join(f"{int(np.median(r[:, k])):6d}" for k in range(4)), f"(n={sel.sum()})")
