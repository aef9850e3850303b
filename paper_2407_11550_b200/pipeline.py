"""Model-level driver: compress every layer after prefill, then decode over the
compressed caches with one CUDA graph per decode step.

Problems are laid out layer-major: problem index = layer * B + request.  All
layers are compressed by ONE adakv_compress call (the prompt caches of every layer
exist once prefill has finished -- the SnapKV/Ada-KV setting),
which lets the per-problem selection clusters of all layers run concurrently.
Decode keeps the model's sequential layer dependence: one adakv_decode launch
per layer per step (fused append + split-K attention + combine), captured once
into a CUDA graph and replayed.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from . import ops


def compress_model(q, k, v, layer_budget, *, kind="ada_snapkv", pool_kernel=7, alpha=0.2, sink_tokens=4,
                   reserve=0, layer_budgets=None, out=None, ws=None, first_layer=0,
                   gather_stream=None) -> ops.CompressedCache:
    """q [L, B, H, m, d]; k, v [L, B, G, n, d] -> one CompressedCache with P = L*B problems.

    first_layer: with `out` (a cache over the whole model), these L layers are the model's
    layers [first_layer, first_layer + L) -- layers compressed in chunks as they arrive.
    gather_stream: see ops.compress (the chunk's gather forked onto that stream)."""
    Lyr, B = q.shape[:2]
    qq = q.reshape(Lyr * B, *q.shape[2:])
    kk = k.reshape(Lyr * B, *k.shape[2:])
    vv = v.reshape(Lyr * B, *v.shape[2:])
    return ops.compress(qq, kk, vv, layer_budget, kind=kind, pool_kernel=pool_kernel, alpha=alpha,
                        sink_tokens=sink_tokens, reserve=reserve, layer_budgets=layer_budgets, out=out, ws=ws,
                        first_problem=first_layer * B, gather_stream=gather_stream)


def pyramid_problem_budgets(avg_outside_per_layer, layers, batch, G, m, beta_max=1.5, beta_min=0.5, device=None):
    """Per-problem layer budgets for compress_model under the pyramid kinds: the linear
    schedule of pyramid_layer_budgets (budget.hpp:169-191) over the layers' OUTSIDE budgets,
    plus the m*G window entries, repeated for every request (problems are layer-major)."""
    sched = ops.pyramid_layer_budgets(int(avg_outside_per_layer), int(layers), float(beta_max), float(beta_min))
    lb = torch.as_tensor(sched, dtype=torch.int64).repeat_interleave(int(batch)) + int(m) * int(G)
    return lb.to(device) if device is not None else lb


def compress_question_agnostic(q_ctx, k_ctx, v_ctx, layer_budget, k_question, v_question, *,
                               kind="ada_snapkv", pool_kernel=7, alpha=0.2, reserve=0, layer_budgets=None):
    """Question-agnostic compression (config 5): the observation window is the
    last m tokens of the CONTEXT (q_ctx = their queries, [L, B, H, m, d]); the context cache
    is compressed first and the question tokens' K/V ([L, B, G, T, d]) are appended afterwards
    with one append_kv of T rows per segment.  `reserve` must cover T plus the decode steps."""
    Lyr, B = q_ctx.shape[:2]
    T = k_question.shape[3]
    if reserve < T:
        raise L.InvalidArgument(1, "compress_question_agnostic: reserve must cover the question tokens")
    cache = compress_model(q_ctx, k_ctx, v_ctx, layer_budget, kind=kind, pool_kernel=pool_kernel, alpha=alpha,
                           reserve=reserve, layer_budgets=layer_budgets)
    G, d = k_question.shape[2], k_question.shape[4]
    ops.append_rows(cache, k_question.reshape(Lyr * B * G, T, d), v_question.reshape(Lyr * B * G, T, d))
    return cache


def decode_layer(lib, c, layer, batch, q, k_new, v_new, out, ws, max_rows, stream, chained, scale=1):
    """adakv_decode of one layer's B*G segments of a model-wide cache (problems layer-major).
    chained: the kernel enqueued just before on `stream` is the decode of another layer
    (ADAKV_DECODE_CHAINED: its cache rows stream in while that one finishes)."""
    G, H, d = c.G, c.H, c.d
    seg = layer * batch * G
    L.check(lib.adakv_decode(
        ops._dt(q), batch, H, G, d, int(scale), C.c_void_p(q.data_ptr()), C.c_void_p(c.k.data_ptr()),
        C.c_void_p(c.v.data_ptr()), c.k.shape[0], C.c_void_p(c.seg_start.data_ptr() + 4 * seg),
        C.c_void_p(c.seg_cap.data_ptr() + 4 * seg), C.c_void_p(c.seqlens.data_ptr() + 4 * seg), int(max_rows),
        None if k_new is None else C.c_void_p(k_new.data_ptr()),
        None if v_new is None else C.c_void_p(v_new.data_ptr()), C.c_void_p(out.data_ptr()),
        C.c_void_p(ws.data_ptr()), ws.numel(), L.DECODE_CHAINED if chained else 0, stream))


class DecodeGraph:
    """One decode step over all layers, captured as a CUDA graph.

    Static device buffers q [L, B, H, d], k_new / v_new [L, B, G, d] and out [L, B, H, d]
    are refreshed by the caller between replays (e.g. copy_ from pinned host memory).
    """

    def __init__(self, cache: ops.CompressedCache, layers: int, batch: int, max_rows: int, scale=True,
                 use_graph=True):
        self.cache = cache
        self.L, self.B = layers, batch
        H, G, d = cache.H, cache.G, cache.d
        dev = cache.k.device
        dt = cache.k.dtype
        self.q = torch.zeros((layers, batch, H, d), dtype=dt, device=dev)
        self.k_new = torch.zeros((layers, batch, G, d), dtype=dt, device=dev)
        self.v_new = torch.zeros((layers, batch, G, d), dtype=dt, device=dev)
        self.out = torch.zeros((layers, batch, H, d), dtype=dt, device=dev)
        self.max_rows = int(max_rows)
        nb = ops.decode_workspace_bytes(batch, H, G, d, self.max_rows)
        self.ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
        self.scale = int(bool(scale))
        self._dt = ops._dt(self.q)
        self._lib = L.lib()
        self.graph = None
        if use_graph:
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream())
            self.graph = torch.cuda.CUDAGraph()
            # capture does not execute: the caches are untouched by capture itself
            with torch.cuda.stream(s):
                with torch.cuda.graph(self.graph, stream=s):
                    self._launch_all()
            torch.cuda.current_stream().wait_stream(s)

    def _launch_all(self):
        c = self.cache
        H, G, d, B = c.H, c.G, c.d, self.B
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for l in range(self.L):
            decode_layer(self._lib, c, l, B, self.q[l], self.k_new[l], self.v_new[l], self.out[l], self.ws,
                         self.max_rows, st, chained=l > 0, scale=self.scale)

    def step(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch_all()
        return self.out


def algorithmic_bytes_compress(L, B, H, G, n_o, m, d, layer_budget, esize=2):
    """e*(G*n_o*d + H*m*d) + 4*e*d*LB per layer per request."""
    return L * B * (esize * (G * n_o * d + H * m * d) + 4 * esize * d * layer_budget)


def algorithmic_bytes_decode_step(L, B, H, G, d, total_rows, esize=2):
    """2*e*d*sum_g len_g + 2*e*H*d + 2*e*G*d per step per layer per request;
    total_rows = sum over all layers/requests/groups of the cache length attended this step."""
    return 2 * esize * d * total_rows + L * B * (2 * esize * H * d + 2 * esize * G * d)
