"""Supplementary bench lines at BASELINE.json configs 3, 4 and 5 (imported by bench.py).

config 3: Mistral-7B shapes (32 Q / 8 KV heads, d = 128, 32 layers), 128K prompt, batch 8,
          per-head budgets 128 / 1024 / 4096; requests batch-sharded over the ranks (8 / N per
          rank, strong scaling).  Each rank compresses its requests layer by layer into one
          model-wide cache (ops.compress first_problem: a layer's prompt KV is consumed as it is
          produced; two synthetic layer inputs alternate, 4.3 GB each, far above L2), then runs
          `steps` decode steps, one launch per layer carrying the rank's requests.
config 4: Llama-3.1-70B shapes (64 Q / 8 KV heads, 80 layers), 64K prompt, per-head budget 2048
          (not given in BASELINE.json), batch 1, KV groups sharded over the ranks
          (8 / N groups per rank) with one all-gather per layer (sharding.py); each layer's
          compress is compress_kv_group_sharded, then `steps` decode steps over the 80 layers.
config 5: Llama-3.1-8B shapes, 32 layers, 32K context, budget 1024/head, question-agnostic
          (window = the context's last 32 tokens, 64 question tokens appended after
          compression), 32 requests batch-sharded over the ranks (4 per GPU on 8 GPUs).
All times are CUDA-event times on the launching stream, max over ranks.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import paper_2407_11550_b200 as A
from paper_2407_11550_b200 import ops
from paper_2407_11550_b200 import pipeline as PL
from paper_2407_11550_b200.synthetic import planted_layer


def _ev():
    return torch.cuda.Event(enable_timing=True)


def _max_over_ranks(x, dev):
    if dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return x


def _decode_graph(lib, caches, layers, batch, qs, ks, vs, outs, ws, max_rows):
    """One CUDA graph: `steps` decode steps x layers, chained within the graph."""
    dev = qs.device
    steps = qs.shape[0]
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream(device=dev)
    st.wait_stream(torch.cuda.current_stream())
    import ctypes as C
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for s in range(steps):
                for l in range(layers):
                    c, li = caches(l)
                    PL.decode_layer(lib, c, li, batch, qs[s, l], ks[s, l], vs[s, l], outs[l], ws, max_rows,
                                    C.c_void_p(st.cuda_stream), chained=s > 0 or l > 0)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    return g


def config3(dev, peak, rank, world, budgets=(128, 1024, 4096), steps=128, reps=2):
    L, B_all, H, G, d, m, n = 32, 8, 32, 8, 128, 32, 131072
    n_o = n - m
    mine = list(range(rank, B_all, world))
    B = len(mine)
    lib = A.lib()
    # two synthetic layer inputs (alternating over the 32 layers), this rank's requests
    inputs = [planted_layer(B, H, G, n_o, m, d, seed=300 + 17 * i + rank, dtype=torch.bfloat16, device=dev)
              for i in range(2)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(900 + rank)
    qs = torch.randn((steps, L, B, H, d), generator=gen, device=dev).to(torch.bfloat16)
    ks = torch.randn((steps, L, B, G, d), generator=gen, device=dev).to(torch.bfloat16)
    vs = torch.randn((steps, L, B, G, d), generator=gen, device=dev).to(torch.bfloat16)
    res = {}
    for b in budgets:
        LB = b * G
        reserve = steps + 1
        P = L * B
        cache = ops.CompressedCache(
            k=torch.empty((P * (LB + G * reserve), d), dtype=torch.bfloat16, device=dev),
            v=torch.empty((P * (LB + G * reserve), d), dtype=torch.bfloat16, device=dev),
            seg_start=torch.empty(P * G, dtype=torch.int32, device=dev),
            seqlens=torch.empty(P * G, dtype=torch.int32, device=dev),
            budgets=torch.empty(P * G, dtype=torch.int32, device=dev), P=P, H=H, G=G, m=m, d=d, reserve=reserve,
            layer_budget=LB, seg_cap=torch.empty(P * G, dtype=torch.int32, device=dev))
        ws = None

        def compress_all():
            for l in range(L):
                q, k, v = inputs[l & 1]
                ops.compress(q, k, v, LB, reserve=reserve, out=cache, first_problem=l * B, ws=ws)

        compress_all()  # warm
        seq0 = cache.seqlens.clone()
        max_rows = int(cache.seg_cap.max())
        outs = torch.empty((L, B, H, d), dtype=torch.bfloat16, device=dev)
        dws = torch.zeros(ops.decode_workspace_bytes(B, H, G, d, max_rows), dtype=torch.uint8, device=dev)
        graph = _decode_graph(lib, lambda l: (cache, l), L, B, qs, ks, vs, outs, dws, max_rows)
        cms, dms = [], []
        for _ in range(reps + 1):
            cache.seqlens.copy_(seq0)
            e0, e1, e2 = _ev(), _ev(), _ev()
            if dist.is_initialized():
                dist.barrier()
            torch.cuda.synchronize()
            e0.record()
            compress_all()
            e1.record()
            graph.replay()
            e2.record()
            torch.cuda.synchronize()
            cms.append(e0.elapsed_time(e1))
            dms.append(e1.elapsed_time(e2))
        cm = _max_over_ranks(float(np.median(cms[1:])), dev)
        dm = _max_over_ranks(float(np.median(dms[1:])), dev)
        bud = cache.budgets.view(P, G).to(torch.int64)
        rows0 = int(bud.sum()) + P * G * m
        bytes_c = world * PL.algorithmic_bytes_compress(L, B, H, G, n_o, m, d, LB)
        rows_total = steps * rows0 + P * G * steps * (steps + 1) // 2
        bytes_d = world * (2 * 2 * d * rows_total + steps * L * B * (2 * 2 * H * d + 2 * 2 * G * d))
        dec_us = dm * 1e3 / (steps * L)
        res[str(b)] = {
            "compress_ms_per_layer": round(cm / L, 4), "compress_gbs": round(bytes_c / (cm * 1e-3) / 1e9, 1),
            "compress_frac": round(bytes_c / (cm * 1e-3) / 1e9 / peak, 4),
            "decode_us_per_launch": round(dec_us, 3), "decode_gbs": round(bytes_d / (dm * 1e-3) / 1e9, 1),
            "decode_frac": round(bytes_d / (dm * 1e-3) / 1e9 / peak, 4),
            "decode_bytes_per_launch": int(bytes_d / world / (steps * L))}
        del cache, graph, dws
        torch.cuda.empty_cache()
    return {"workload": f"Mistral-7B shapes, 32 layers, 128K prompt, batch 8 ({B} per rank x {world} ranks), "
                        f"compress all layers + {steps} decode steps (one launch per layer, {B} requests)",
            "scaling": "strong (8 requests split over the ranks)", "budgets": res}


def config4(dev, peak, rank, world, steps=64, reps=2, layers=80):
    H, G, d, m, n, budget = 64, 8, 128, 32, 65536, 2048
    n_o = n - m
    if G % world:
        return {"skipped": f"{G} KV groups do not split over {world} ranks"}
    Gl, Hl = G // world, H // world
    g0 = rank * Gl
    LB = budget * G
    lib = A.lib()
    group = dist.group.WORLD if dist.is_initialized() else None
    # this rank's groups of two synthetic layer inputs (alternating over the 80 layers)
    inputs = []
    for i in range(2):
        q, k, v = planted_layer(1, H, G, n_o, m, d, seed=400 + i, dtype=torch.bfloat16, device=dev)
        inputs.append((q[0, g0 * (H // G):(g0 + Gl) * (H // G)].contiguous(), k[0, g0:g0 + Gl].contiguous(),
                       v[0, g0:g0 + Gl].contiguous()))
        del q, k, v
    reserve = steps + 1
    from paper_2407_11550_b200.sharding import compress_kv_group_sharded

    def compress_all():
        out, nbytes = [], 0
        for l in range(layers):
            q, k, v = inputs[l & 1]
            c, a = compress_kv_group_sharded(q, k, v, LB, G, g0=g0, group=group, reserve=reserve)
            out.append(c)
            nbytes = a.payload_bytes
        return out, nbytes

    caches, payload = compress_all()  # warm (allocates every workspace outside the capture)
    # the 80 layers' sharded compress (scores, local top-k, the all-gather, the merge, the
    # gather) is one CUDA graph: about fifteen launches per layer, none of them host-synchronised
    cgraph = torch.cuda.CUDAGraph()
    cst = torch.cuda.Stream(device=dev)
    cst.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cst):
        with torch.cuda.graph(cgraph, stream=cst):
            fresh, _ = compress_all()
    torch.cuda.current_stream().wait_stream(cst)
    torch.cuda.synchronize()
    gen = torch.Generator(device=dev)
    gen.manual_seed(950 + rank)
    qs = torch.randn((steps, layers, 1, Hl, d), generator=gen, device=dev).to(torch.bfloat16)
    ks = torch.randn((steps, layers, 1, Gl, d), generator=gen, device=dev).to(torch.bfloat16)
    vs = torch.randn((steps, layers, 1, Gl, d), generator=gen, device=dev).to(torch.bfloat16)
    max_rows = max(int(c.seg_cap.max()) for c in caches)
    outs = torch.empty((layers, 1, Hl, d), dtype=torch.bfloat16, device=dev)
    dws = torch.zeros(ops.decode_workspace_bytes(1, Hl, Gl, d, max_rows), dtype=torch.uint8, device=dev)
    cms, dms = [], []
    seq0 = [c.seqlens.clone() for c in caches]
    graph = _decode_graph(lib, lambda l: (caches[l], 0), layers, 1, qs, ks, vs, outs, dws, max_rows)
    for _ in range(reps + 1):
        for c, s0 in zip(caches, seq0):
            c.seqlens.copy_(s0)
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1, e2 = _ev(), _ev(), _ev()
        e0.record()
        cgraph.replay()
        e1.record()
        graph.replay()  # over the warm-up caches (same shapes and budgets: identical inputs)
        e2.record()
        torch.cuda.synchronize()
        cms.append(e0.elapsed_time(e1))
        dms.append(e1.elapsed_time(e2))
    cm = _max_over_ranks(float(np.median(cms[1:])), dev)
    dm = _max_over_ranks(float(np.median(dms[1:])), dev)
    rows0 = sum(int(c.seqlens.sum()) for c in caches) - layers * Gl * steps  # after the replays' appends
    bytes_c = layers * (2 * (G * n_o * d + H * m * d) + 4 * 2 * d * LB)  # whole model, all ranks
    rows_total = steps * rows0 + layers * Gl * steps * (steps + 1) // 2
    bytes_d_rank = 2 * 2 * d * rows_total + steps * layers * (2 * 2 * Hl * d + 2 * 2 * Gl * d)
    return {"workload": f"Llama-3.1-70B shapes, {layers} layers, 64K prompt, budget {budget}/head, batch 1, "
                        f"KV groups sharded {Gl} per rank x {world} ranks, one all-gather per layer "
                        f"({payload} B per rank), {steps} decode steps",
            "scaling": "strong (the 8 KV groups split over the ranks)",
            "compress_ms_per_layer": round(cm / layers, 4), "compress_gbs": round(bytes_c / (cm * 1e-3) / 1e9, 1),
            "compress_frac": round(bytes_c / (cm * 1e-3) / 1e9 / peak, 4),
            "decode_us_per_launch": round(dm * 1e3 / (steps * layers), 3),
            "decode_gbs_per_rank": round(bytes_d_rank / (dm * 1e-3) / 1e9, 1),
            "decode_frac": round(bytes_d_rank / (dm * 1e-3) / 1e9 / peak, 4)}


def config5(dev, peak, rank, world, steps=64, reps=2, T=64):
    """Config 5: question-agnostic compression -- Llama-3.1-8B shapes, 32
    layers, 32K context, budget 1024/head, 32 requests batch-sharded over the ranks (4 per GPU on
    8 GPUs).  Per layer the window is the context's last 32 tokens; after compression the T
    question tokens are appended to every segment (append_rows), then `steps` decode steps."""
    L, B_all, H, G, d, m, n, budget = 32, 32, 32, 8, 128, 32, 32768, 1024
    n_o = n - m
    mine = list(range(rank, B_all, world))
    B = len(mine)
    lib = A.lib()
    inputs = [planted_layer(B, H, G, n_o, m, d, seed=500 + 13 * i + rank, dtype=torch.bfloat16, device=dev)
              for i in range(2)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(990 + rank)
    kq = torch.randn((B * G, T, d), generator=gen, device=dev).to(torch.bfloat16)
    vq = torch.randn((B * G, T, d), generator=gen, device=dev).to(torch.bfloat16)
    qs = torch.randn((steps, L, B, H, d), generator=gen, device=dev).to(torch.bfloat16)
    ks = torch.randn((steps, L, B, G, d), generator=gen, device=dev).to(torch.bfloat16)
    vs = torch.randn((steps, L, B, G, d), generator=gen, device=dev).to(torch.bfloat16)
    LB = budget * G
    reserve = T + steps + 1
    P = L * B
    cache = ops.CompressedCache(
        k=torch.empty((P * (LB + G * reserve), d), dtype=torch.bfloat16, device=dev),
        v=torch.empty((P * (LB + G * reserve), d), dtype=torch.bfloat16, device=dev),
        seg_start=torch.empty(P * G, dtype=torch.int32, device=dev),
        seqlens=torch.empty(P * G, dtype=torch.int32, device=dev),
        budgets=torch.empty(P * G, dtype=torch.int32, device=dev), P=P, H=H, G=G, m=m, d=d, reserve=reserve,
        layer_budget=LB, seg_cap=torch.empty(P * G, dtype=torch.int32, device=dev))

    def compress_all():
        for l in range(L):
            q, k, v = inputs[l & 1]
            ops.compress(q, k, v, LB, reserve=reserve, out=cache, first_problem=l * B)
        # the question tokens after compression: every layer's segments get the same T rows here
        for l in range(L):
            sub = ops.CompressedCache(k=cache.k, v=cache.v, seg_start=cache.seg_start[l * B * G:(l + 1) * B * G],
                                      seqlens=cache.seqlens[l * B * G:(l + 1) * B * G], budgets=cache.budgets,
                                      P=B, H=H, G=G, m=m, d=d, reserve=reserve, layer_budget=LB,
                                      seg_cap=cache.seg_cap[l * B * G:(l + 1) * B * G])
            ops.append_rows(sub, kq, vq, check=False)

    compress_all()
    seq_q = cache.seqlens.clone()
    max_rows = int(cache.seg_cap.max())
    outs = torch.empty((L, B, H, d), dtype=torch.bfloat16, device=dev)
    dws = torch.zeros(ops.decode_workspace_bytes(B, H, G, d, max_rows), dtype=torch.uint8, device=dev)
    graph = _decode_graph(lib, lambda l: (cache, l), L, B, qs, ks, vs, outs, dws, max_rows)
    cms, dms = [], []
    for _ in range(reps + 1):
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1, e2 = _ev(), _ev(), _ev()
        e0.record()
        compress_all()
        e1.record()
        cache.seqlens.copy_(seq_q)
        graph.replay()
        e2.record()
        torch.cuda.synchronize()
        cms.append(e0.elapsed_time(e1))
        dms.append(e1.elapsed_time(e2))
    cm = _max_over_ranks(float(np.median(cms[1:])), dev)
    dm = _max_over_ranks(float(np.median(dms[1:])), dev)
    rows0 = int(seq_q.to(torch.int64).sum())
    bytes_c = world * (PL.algorithmic_bytes_compress(L, B, H, G, n_o, m, d, LB) + L * B * G * T * 2 * 2 * d * 2)
    rows_total = steps * rows0 + P * G * steps * (steps + 1) // 2
    bytes_d = world * (2 * 2 * d * rows_total + steps * L * B * (2 * 2 * H * d + 2 * 2 * G * d))
    return {"workload": f"Llama-3.1-8B shapes, 32 layers, 32K context, budget {budget}/head, question-agnostic "
                        f"(window = last 32 context tokens, {T} question tokens appended after compression), "
                        f"32 requests ({B} per rank x {world} ranks), {steps} decode steps",
            "scaling": "strong (32 requests split over the ranks)",
            "compress_ms_per_layer": round(cm / L, 4), "compress_gbs": round(bytes_c / (cm * 1e-3) / 1e9, 1),
            "compress_frac": round(bytes_c / (cm * 1e-3) / 1e9 / peak, 4),
            "decode_us_per_launch": round(dm * 1e3 / (steps * L), 3),
            "decode_gbs": round(bytes_d / (dm * 1e-3) / 1e9, 1), "decode_frac": round(bytes_d / (dm * 1e-3) / 1e9 / peak, 4)}
