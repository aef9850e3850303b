"""Per-stage device timing (CUDA graphs, CUDA events on the capture stream).

    python scripts/kbench.py [--layers 32] [--prompt 32768]
Prints one JSON line per stage: window scoring (K1), full compress, decode step.
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200 import pipeline as PL  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402


def graph_time(fn, iters=10, warm=3):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--prompt", type=int, default=32768)
    ap.add_argument("--generic", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    L = A.lib()
    if args.generic:
        L.adakv_set_tensor_core_scoring(0)
    P, H, G, m, d = args.layers, 32, 8, 32, 128
    n = args.prompt
    n_o = n - m
    LB = 2048 * G
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=11, dtype=torch.bfloat16, device=dev)
    peak = 6531.0  # MEASURED_PEAKS.json hbm_gbs
    out = {}
    # K1 alone
    gs = torch.empty((P, G, n_o), dtype=torch.float32, device=dev)
    shape = A.ops.layer_shape(P, H, G, m, n_o, d)
    nb = C.c_size_t()
    A._lib.check(L.adakv_window_scores_workspace(2, C.byref(shape), C.byref(nb)))
    ws = torch.zeros(nb.value * 2, dtype=torch.uint8, device=dev)

    def k1():
        A._lib.check(L.adakv_window_scores(2, C.byref(shape), 7, 1, C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                           None, C.c_void_p(gs.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(),
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    t = graph_time(k1)
    bytes_k1 = P * 2 * (G * n_o * d + H * m * d)
    out["score_ms_per_layer"] = t / P
    out["score_gbs"] = bytes_k1 / (t * 1e-3) / 1e9
    out["score_frac"] = out["score_gbs"] / peak
    # full compress
    cache = A.compress(q, k, v, LB, reserve=8)
    cws = A.ops.workspace(0, dev, "compress")
    t = graph_time(lambda: A.compress(q, k, v, LB, reserve=8, out=cache, ws=cws))
    bytes_c = PL.algorithmic_bytes_compress(P, 1, H, G, n_o, m, d, LB)
    out["compress_ms_per_layer"] = t / P
    out["compress_gbs"] = bytes_c / (t * 1e-3) / 1e9
    out["compress_frac"] = out["compress_gbs"] / peak
    # the same compress as 4 calls of P/4 layers (a prefill compressed as its layers arrive),
    # with and without each chunk's gather forked onto a second stream (adakv_compress_split)
    if P % 4 == 0 and not args.generic:
        nch, lc = 4, P // 4
        gst = torch.cuda.Stream()
        wss = [torch.zeros(A.ops.compress_workspace_bytes(q[:lc], k[:lc]), dtype=torch.uint8, device=dev)
               for _ in range(2)]
        evs = [torch.cuda.Event(), torch.cuda.Event()]

        def chunked(split):
            cur = torch.cuda.current_stream()
            if split:
                gst.wait_stream(cur)
            for c in range(nch):
                if split and c >= 2:
                    cur.wait_event(evs[c & 1])
                sl = slice(c * lc, (c + 1) * lc)
                A.compress(q[sl], k[sl], v[sl], LB, reserve=8, out=cache, ws=wss[c & 1], first_problem=c * lc,
                           gather_stream=gst if split else None)
                if split:
                    evs[c & 1].record(gst)
            if split:
                cur.wait_stream(gst)
        out["compress_4chunks_ms_per_layer"] = graph_time(lambda: chunked(False)) / P
        out["compress_4chunks_split_gather_ms_per_layer"] = graph_time(lambda: chunked(True)) / P
    # select alone (scores already computed) -- via segmented_select on fp32 scores
    sc = gs.reshape(P, G * n_o)
    import numpy as np
    off = np.arange(G + 1) * n_o
    t = graph_time(lambda: A.segmented_select(sc, off, LB - m * G, "adaptive", blend=True, alpha=0.2, repair=True,
                                              want_keep=False))
    out["select_us_per_call"] = t * 1e3
    # layout + gather alone (the compaction: 4 e d LB bytes per layer)
    r = A.segmented_select(sc, off, LB - m * G, "adaptive", blend=True, alpha=0.2, repair=True, want_keep=False)
    bud, kp = r["budgets"].contiguous(), r["kept_pos"]
    gk = torch.empty_like(cache.k)
    gv = torch.empty_like(cache.v)
    gss, gsl, gcap = (torch.empty(P * G, dtype=torch.int32, device=dev) for _ in range(3))

    def gather():
        A._lib.check(L.adakv_gather(2, C.byref(shape), LB, None, C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                    C.c_void_p(bud.data_ptr()), C.c_void_p(kp.data_ptr()), kp.shape[1], 8,
                                    C.c_void_p(gk.data_ptr()), C.c_void_p(gv.data_ptr()), C.c_void_p(gss.data_ptr()),
                                    C.c_void_p(gsl.data_ptr()), C.c_void_p(gcap.data_ptr()), None,
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    t = graph_time(gather)
    out["gather_us_per_layer"] = t * 1e3 / P
    out["gather_gbs"] = P * 4 * 2 * d * LB / (t * 1e-3) / 1e9
    # decode: one step over all P layers (P launches, sequential), no append
    torch.cuda.synchronize()
    budgets = cache.budgets.cpu()
    max_rows = int(budgets.max()) + m + 16
    dg = PL.DecodeGraph(cache, P, 1, max_rows, use_graph=False)
    dg.q.normal_()

    def dec():
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for l in range(P):
            PL.decode_layer(L, cache, l, 1, dg.q[l], None, None, dg.out[l], dg.ws, max_rows, stream, chained=l > 0)
    t = graph_time(dec, iters=20)
    rows = int(budgets.sum()) + P * G * m
    bytes_d = PL.algorithmic_bytes_decode_step(P, 1, H, G, d, rows)
    out["decode_us_per_layer_step"] = t * 1e3 / P
    out["decode_gbs"] = bytes_d / (t * 1e-3) / 1e9
    out["decode_frac"] = out["decode_gbs"] / peak
    out["config"] = dict(layers=P, prompt=n, layer_budget=LB, generic=args.generic)
    print(json.dumps({k_: (round(v_, 4) if isinstance(v_, float) else v_) for k_, v_ in out.items()}), flush=True)


if __name__ == "__main__":
    main()
