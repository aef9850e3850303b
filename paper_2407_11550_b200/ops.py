"""torch-tensor front end over the C ABI (include/adakv_b200.h).

Every function launches on torch's current CUDA stream and calls straight into
lib/libadakv_b200.so; nothing here computes on the CPU.  Names follow the
reference (adakv::evict_layer, window_scores, adaptive_allocation, ...), see
the C header for the file:line each entry point replaces.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

_DT = {torch.bfloat16: L.BF16, torch.float32: L.F32, torch.float64: L.F64}


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise L.InvalidArgument(1, f"unsupported dtype {t.dtype}") from None


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise L.InvalidArgument(1, "tensors must live on a CUDA device (no CPU path)")
        if t is not None and not t.is_contiguous():
            raise L.InvalidArgument(1, "tensors must be contiguous")


_ws_cache: dict = {}


def workspace(nbytes: int, device, key="default") -> torch.Tensor:
    """Cached uint8 workspace (zero-initialised on first allocation), one per (device, stream,
    purpose): calls issued on different streams never share scratch.  A workspace returned by
    an op is valid until the next op of the same purpose on the same stream."""
    k = (str(device), torch.cuda.current_stream(device).cuda_stream, key)
    t = _ws_cache.get(k)
    if t is None or t.numel() < nbytes:
        t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[k] = t
    return t


def policy_config(kind="ada_snapkv", pool_kernel=7, alpha=0.2, sink_tokens=4, gqa_group_size=1,
                  scale=True, window_size=32) -> L.PolicyConfig:
    return L.PolicyConfig(L.KINDS[kind] if isinstance(kind, str) else int(kind), int(bool(scale)),
                          int(window_size), int(pool_kernel), float(alpha), int(sink_tokens),
                          int(gqa_group_size))


def layer_shape(P, H, G, m, n_o, d) -> L.LayerShape:
    return L.LayerShape(int(P), int(H), int(G), int(m), int(n_o), int(d))


@dataclass
class CompressedCache:
    """The flattened variable-length cache (flat_cache.hpp:24-36) on the device.

    Segment (p, g) holds rows [seg_start, seg_start + seqlens) of k/v: kept outside
    rows in original order, then the m window rows (policies.hpp:273-290);
    capacity per segment = budgets + m + reserve (seg_cap); decode and append never write
    past it (ERR_CAPACITY, raised by workspace_status).
    """
    k: torch.Tensor
    v: torch.Tensor
    seg_start: torch.Tensor  # int32 [P*G]
    seqlens: torch.Tensor    # int32 [P*G]
    budgets: torch.Tensor    # int32 [P*G] outside budget per group (BudgetAllocation)
    P: int
    H: int
    G: int
    m: int
    d: int
    reserve: int
    layer_budget: int
    scores: torch.Tensor | None = None  # [P, G, n_o] pooled group scores
    keep: torch.Tensor | None = None    # uint8 [P, G, n_o] decision
    seg_cap: torch.Tensor | None = None  # int32 [P*G] capacity in rows (derived if not given)

    def __post_init__(self):
        if self.seg_cap is None:
            # a hand-built cache of back-to-back segments: each runs to the next one's start
            # (the last to the end of the planes)
            st = self.seg_start.to(torch.int64)
            if st.numel():
                order = torch.argsort(st)
                ends = torch.empty_like(st)
                ends[order] = torch.cat([st[order][1:], st.new_tensor([self.k.shape[0]])])
                self.seg_cap = (ends - st).to(torch.int32)
            else:
                self.seg_cap = self.seg_start.clone()

    @property
    def max_rows(self) -> int:
        """Upper bound of any segment's length: its largest capacity (seqlens <= seg_cap always).
        Read from the device once (one synchronisation) and cached."""
        if getattr(self, "_max_rows", None) is None:
            self._max_rows = int(self.seg_cap.max()) if self.seg_cap.numel() else 1
        return self._max_rows

    def segment(self, p: int, g: int):
        s = int(self.seg_start[p * self.G + g])
        n = int(self.seqlens[p * self.G + g])
        return self.k[s:s + n], self.v[s:s + n]


def host_device_pointer(t: torch.Tensor) -> C.c_void_p:
    """Device address of a pinned, contiguous CPU tensor (adakv_host_device_pointer)."""
    if t.is_cuda or not t.is_pinned():
        raise L.InvalidArgument(1, "host buffers must be pinned CPU tensors (tensor.pin_memory())")
    if not t.is_contiguous():
        raise L.InvalidArgument(1, "tensors must be contiguous")
    dp = C.c_void_p()
    L.check(L.lib().adakv_host_device_pointer(C.c_void_p(t.data_ptr()), C.byref(dp)))
    return dp


def compress(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layer_budget: int, kind="ada_snapkv",
             pool_kernel=7, alpha=0.2, sink_tokens=4, scale=True, reserve=0, layer_budgets=None,
             return_scores=False, return_keep=False, out: CompressedCache | None = None,
             ws: torch.Tensor | None = None, first_problem: int = 0, validate=False, check=False,
             gather_stream: torch.cuda.Stream | None = None) -> CompressedCache:
    """evict_layer (policies.hpp:204-293) for P problems at once.

    q [P, H, m, d]; k, v [P, G, n, d] with the observation window in the last m rows.
    v may be a pinned CPU tensor: only the retained and window rows (layer_budget per
    problem) are then read, by the gather, straight from host memory.
    layer_budget counts unique KV entries per problem, window included.
    layer_budgets: optional int64 CUDA tensor [P] (per-problem budgets, pyramid kinds).
    first_problem: with `out` and uniform budgets, write these P problems as problems
    [first_problem, first_problem + P) of `out` (a model's layers compressed in chunks, e.g. as
    their inputs arrive); the rows land exactly where one call over all problems puts them.
    validate: also scan every K and V entry for NaN/Inf (LayerCache::validate,
    attention.hpp:76-83; adakv_validate_finite).  Without it the device still latches the
    non-finite entries that reach the window statistics or the copied rows.
    check: synchronise and raise the reference's exception for anything the device latched
    (non-finite input, per-problem budget below the floor / above the capacity).
    gather_stream: run the final gather (the copy of the retained rows into out.k / out.v) on
    this stream, forked after the selection (adakv_compress_split): the current stream goes on
    at once, so a model compressed in chunks overlaps chunk i's gather with chunk i+1's scoring.
    The caller must make the cache's readers wait for gather_stream, and must not reuse `ws`
    on the current stream before that (the gather reads it).
    """
    _need_cuda(q, k)
    if v.is_cuda:
        _need_cuda(v)
        v_ptr = _p(v)
    else:
        v_ptr = host_device_pointer(v)
    P, H, m, d = q.shape
    P2, G, n, d2 = k.shape
    if P2 != P or d2 != d or v.shape != k.shape or k.dtype != q.dtype or v.dtype != q.dtype:
        raise L.InvalidArgument(1, "compress: q/k/v shape or dtype mismatch")
    n_o = n - m
    dt = _dt(q)
    shape = layer_shape(P, H, G, m, n_o, d)
    cfg = policy_config(kind, pool_kernel, alpha, sink_tokens, H // G if G else 1, scale, m)
    lib = L.lib()
    if layer_budgets is not None:
        lb_host = layer_budgets.detach().cpu().numpy().astype(np.int64)
        # evict_layer's floor and apportion's capacity per problem (policies.hpp:229-231,
        # budget.hpp:48-59); the device latches the same errors for direct C-ABI callers
        if lb_host.size and int(lb_host.min()) < m * G + G:
            raise L.InvalidArgument(1, "evict_layer: budget below the window-plus-one floor")
        if lb_host.size and int(lb_host.max()) - m * G > G * n_o:
            raise L.InvalidArgument(1, "apportion: total exceeds capacity")
        rows = int(lb_host.sum()) + P * G * reserve
        lbmax = int(lb_host.max()) if lb_host.size else 0
    else:
        rows = P * (layer_budget + G * reserve)
        lbmax = layer_budget
    dev = q.device
    acc_dtype = torch.float64 if q.dtype == torch.float64 else torch.float32
    if out is None:
        out = CompressedCache(
            k=torch.empty((max(rows, 1), d), dtype=q.dtype, device=dev),
            v=torch.empty((max(rows, 1), d), dtype=q.dtype, device=dev),
            seg_start=torch.empty(P * G, dtype=torch.int32, device=dev),
            seqlens=torch.empty(P * G, dtype=torch.int32, device=dev),
            seg_cap=torch.empty(P * G, dtype=torch.int32, device=dev),
            budgets=torch.empty(P * G, dtype=torch.int32, device=dev),
            P=P, H=H, G=G, m=m, d=d, reserve=reserve, layer_budget=lbmax,
            scores=torch.empty((P, G, n_o), dtype=acc_dtype, device=dev) if return_scores else None,
            keep=torch.empty((P, G, n_o), dtype=torch.uint8, device=dev) if return_keep else None)
    p0 = int(first_problem)
    row0 = 0
    if p0:
        if out is None or layer_budgets is not None or p0 < 0 or p0 + P > out.P:
            raise L.InvalidArgument(1, "compress: first_problem needs `out` with room and uniform budgets")
        row0 = p0 * (layer_budget + G * reserve)

    def at(t, off):
        return None if t is None else C.c_void_p(t.data_ptr() + off * t.element_size())

    nbytes = C.c_size_t()
    L.check(lib.adakv_compress_workspace(dt, C.byref(shape), C.byref(cfg), C.byref(nbytes)))
    if ws is None:
        ws = workspace(nbytes.value, dev, "compress")
    args = (dt, C.byref(shape), C.byref(cfg), int(layer_budget), _p(layer_budgets), _p(q), _p(k), v_ptr, int(reserve),
            at(out.k, row0 * d), at(out.v, row0 * d), at(out.seg_start, p0 * G), at(out.seqlens, p0 * G),
            at(out.seg_cap, p0 * G), at(out.budgets, p0 * G), at(out.scores, p0 * G * n_o), at(out.keep, p0 * G * n_o),
            _p(ws), ws.numel(), _stream())
    if gather_stream is not None:
        if check:
            raise L.InvalidArgument(1, "compress: check needs the gather on the current stream")
        L.check(lib.adakv_compress_split(*args, C.c_void_p(gather_stream.cuda_stream)))
    else:
        L.check(lib.adakv_compress(*args))
    if row0:  # the library laid the segments out from row 0 of the planes it was given
        if gather_stream is not None:  # after the forked gather has read them
            with torch.cuda.stream(gather_stream):
                out.seg_start[p0 * G:(p0 + P) * G] += row0
        else:
            out.seg_start[p0 * G:(p0 + P) * G] += row0
    out._max_rows = None  # capacities were rewritten
    if validate:
        validate_finite(k, ws)
        validate_finite(v, ws)
    if check:
        workspace_status(ws)
    return out


def compress_workspace_bytes(q: torch.Tensor, k: torch.Tensor, kind="ada_snapkv", pool_kernel=7, alpha=0.2,
                             sink_tokens=4, scale=True) -> int:
    """Workspace bytes of one compress call on inputs shaped like q [P, H, m, d], k [P, G, n, d]
    (e.g. to give each in-flight chunk of a split-gather pipeline its own workspace)."""
    P, H, m, d = q.shape
    G, n = k.shape[1], k.shape[2]
    shape = layer_shape(P, H, G, m, n - m, d)
    cfg = policy_config(kind, pool_kernel, alpha, sink_tokens, H // G if G else 1, scale, m)
    nbytes = C.c_size_t()
    L.check(L.lib().adakv_compress_workspace(_dt(q), C.byref(shape), C.byref(cfg), C.byref(nbytes)))
    return nbytes.value


def validate_finite(x: torch.Tensor, ws: torch.Tensor) -> None:
    """LayerCache::validate (attention.hpp:76-83) on the device: latches a non-finite entry of x
    (device or pinned host tensor) into ws's error word (raised by workspace_status)."""
    ptr = _p(x) if x.is_cuda else host_device_pointer(x)
    L.check(L.lib().adakv_validate_finite(_dt(x), ptr, x.numel(), _p(ws), _stream()))


def window_scores(q: torch.Tensor, k: torch.Tensor, pool_kernel=7, scale=True, head_scores=False,
                  ws: torch.Tensor | None = None):
    """window_scores (policies.hpp:119-132) for every head + group_mean_scores (136-156).

    q [P, H, m, d]; k [P, G, n, d] (outside keys are rows [0, n - m)).
    Returns group scores [P, G, n_o] (and per-head scores [P, H, n_o] if asked).
    """
    _need_cuda(q, k)
    P, H, m, d = q.shape
    _, G, n, _ = k.shape
    n_o = n - m
    dt = _dt(q)
    shape = layer_shape(P, H, G, m, n_o, d)
    acc = torch.float64 if q.dtype == torch.float64 else torch.float32
    gs = torch.empty((P, G, n_o), dtype=acc, device=q.device)
    hs = torch.empty((P, H, n_o), dtype=acc, device=q.device) if head_scores else None
    lib = L.lib()
    nbytes = C.c_size_t()
    L.check(lib.adakv_window_scores_workspace(dt, C.byref(shape), C.byref(nbytes)))
    if ws is None:
        ws = workspace(nbytes.value * 2, q.device, "scores")
    L.check(lib.adakv_window_scores(dt, C.byref(shape), int(pool_kernel), int(bool(scale)), _p(q), _p(k), _p(hs),
                                    _p(gs), _p(ws), ws.numel(), _stream()))
    return (gs, hs) if head_scores else gs


def segmented_select(scores: torch.Tensor, seg_off, total=0, mode="adaptive", blend=False, alpha=1.0,
                     repair=False, streaming=False, sink_tokens=4, budgets: torch.Tensor | None = None,
                     totals: torch.Tensor | None = None, want_keep=True, want_pos=True, want_raw=False):
    """Layer-wide / per-segment selection (budget.hpp:118-158, policies.hpp:80-93, 159-196).

    scores [P, N] f32 or f64 (N = seg_off[-1]); segments are ragged.
    mode: "adaptive" (Algorithm 1), "uniform", or "given" (per-segment top-k with `budgets`).
    Returns dict(budgets int32 [P,S], keep uint8 [P,N], kept_pos int32 [P, stride], raw int32 [P,S]).
    """
    _need_cuda(scores)
    if scores.dtype not in (torch.float32, torch.float64):
        raise L.InvalidArgument(1, "segmented_select: scores must be f32 or f64")
    P, N = scores.shape
    off = np.ascontiguousarray(np.asarray(seg_off, dtype=np.int64))
    S = off.size - 1
    if S > 0 and int(off[-1]) != N:
        raise L.InvalidArgument(1, "segmented_select: seg_off[-1] != N")
    dev = scores.device
    mode_i = {"adaptive": L.ALLOC_ADAPTIVE, "uniform": L.ALLOC_UNIFORM, "given": L.ALLOC_GIVEN}[mode]
    if budgets is None:
        budgets = torch.empty((P, max(S, 1)), dtype=torch.int32, device=dev)
    stride = N if (mode_i == L.ALLOC_GIVEN or totals is not None) else int(total)
    stride = max(stride, 1)
    keep = torch.empty((P, max(N, 1)), dtype=torch.uint8, device=dev) if want_keep else None
    pos = torch.empty((P, stride), dtype=torch.int32, device=dev) if want_pos else None
    raw = torch.empty((P, max(S, 1)), dtype=torch.int32, device=dev) if want_raw else None
    cfg = L.SelectConfig(mode_i, int(bool(blend)), int(bool(repair)), int(bool(streaming)), float(alpha),
                         int(sink_tokens))
    lib = L.lib()
    nbytes = C.c_size_t()
    L.check(lib.adakv_segmented_select_workspace(P, S, C.byref(nbytes)))
    ws = workspace(nbytes.value, dev, "select")
    L.check(lib.adakv_segmented_select(L.F64 if scores.dtype == torch.float64 else L.F32, P, S,
                                       off.ctypes.data_as(L.PI64), _p(scores), int(total), _p(totals),
                                       C.byref(cfg), _p(raw), _p(budgets), _p(keep), _p(pos), stride, _p(ws),
                                       ws.numel(), _stream()))
    return {"budgets": budgets[:, :S], "keep": None if keep is None else keep[:, :N], "kept_pos": pos,
            "raw": None if raw is None else raw[:, :S], "ws": ws}


def workspace_status(ws: torch.Tensor) -> None:
    """Raises the reference's exception if a device-side check latched an error."""
    L.check(L.lib().adakv_workspace_status(_p(ws), _stream()))


def decode_workspace_bytes(P, H, G, d, max_rows) -> int:
    nbytes = C.c_size_t()
    L.check(L.lib().adakv_decode_workspace(P, H, G, d, max_rows, C.byref(nbytes)))
    return nbytes.value


def decode(q: torch.Tensor, cache: CompressedCache, k_new: torch.Tensor | None = None,
           v_new: torch.Tensor | None = None, scale=True, max_rows: int | None = None,
           out: torch.Tensor | None = None, ws: torch.Tensor | None = None, check=False) -> torch.Tensor:
    """One decode step over the compressed cache (attention.hpp:169-196, report.hpp:133-144),
    with append_kv (attention.hpp:126-134) of (k_new, v_new) [P, G, d] fused in.

    q [P, H, d] -> out [P, H, d].  `ws` must be zero-initialised before first use
    (the kernel keeps its tickets re-armed), e.g. torch.zeros(decode_workspace_bytes(...)).
    A segment already at capacity is not appended to; check=True synchronises and raises
    append_kv's InvalidArgument for it (otherwise read it later with workspace_status(ws)).
    """
    _need_cuda(q, k_new, v_new)
    P, H, d = q.shape
    mr = int(max_rows if max_rows is not None else cache.max_rows)
    if out is None:
        out = torch.empty_like(q)
    lib = L.lib()
    if ws is None:
        # the split-K kernels keep per-segment tickets in the workspace and re-arm them, so a
        # workspace is reusable only by calls of the same layout: one cached workspace per
        # (problems, heads, groups, d, max_rows), zeroed when first created
        ws = workspace(decode_workspace_bytes(P, H, cache.G, d, mr), q.device, ("decode", P, H, cache.G, d, mr))
    L.check(lib.adakv_decode(_dt(q), P, H, cache.G, d, int(bool(scale)), _p(q), _p(cache.k), _p(cache.v),
                             cache.k.shape[0], _p(cache.seg_start), _p(cache.seg_cap), _p(cache.seqlens), mr,
                             _p(k_new), _p(v_new), _p(out), _p(ws), ws.numel(), 0, _stream()))
    if check:
        workspace_status(ws)
    return out


def append_kv(cache: CompressedCache, k_new: torch.Tensor, v_new: torch.Tensor, check=True) -> None:
    """append_kv (attention.hpp:126-134) for every segment: k_new/v_new [P*G, d].  A segment at
    capacity is left untouched and (check=True) InvalidArgument is raised, as the reference
    throws on a bad append (attention.hpp:128-131)."""
    append_rows(cache, k_new.contiguous().reshape(k_new.shape[0], 1, -1),
                v_new.contiguous().reshape(v_new.shape[0], 1, -1), check=check)


def append_rows(cache: CompressedCache, k_new: torch.Tensor, v_new: torch.Tensor, check=True) -> None:
    """append_kv (attention.hpp:126-134) of T rows per segment: k_new/v_new [P*G, T, d] (e.g. the
    question tokens after a question-agnostic compression).  The cache needs T spare rows per
    segment (compress(..., reserve >= T + decode steps)); segments without them are left
    untouched and (check=True) InvalidArgument("append_kv: capacity exhausted") is raised."""
    k_new, v_new = k_new.contiguous(), v_new.contiguous()
    _need_cuda(k_new, v_new)
    S, T, d = k_new.shape
    if S != cache.P * cache.G or d != cache.d or v_new.shape != k_new.shape:
        raise L.InvalidArgument(1, "append_kv: row shape mismatch")
    ws = workspace(256, k_new.device, "append")
    if check:
        L.check(L.lib().adakv_clear_workspace_status(_p(ws), _stream()))
    L.check(L.lib().adakv_append_rows(_dt(k_new), S, T, d, _p(cache.k), _p(cache.v), _p(cache.seg_start),
                                      _p(cache.seg_cap), _p(cache.seqlens), _p(k_new.contiguous()),
                                      _p(v_new.contiguous()), _p(ws), _stream()))
    if check:
        workspace_status(ws)


# ---------------------------------------------------------------- budget helpers (device fp64)
def _i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def apportion(quotas, total, caps=None):
    q = np.ascontiguousarray(np.asarray(quotas, np.float64))
    out = np.zeros(max(q.size, 1), np.int64)
    c = None if caps is None else _i64(caps)
    L.check(L.lib().adakv_apportion(_ptr(q), q.size, int(total), _ptr(c), _ptr(out)))
    return out[:q.size]


def uniform_allocation(total, h, caps=None):
    out = np.zeros(max(int(h), 1), np.int64)
    c = None if caps is None else _i64(caps)
    L.check(L.lib().adakv_uniform_allocation(int(total), int(h), _ptr(c), _ptr(out)))
    return out[:int(h)]


def safeguard_blend(adaptive, total, h, alpha, caps=None, adaptive_total=None):
    a = _i64(adaptive)
    out = np.zeros(max(int(h), 1), np.int64)
    c = None if caps is None else _i64(caps)
    at = total if adaptive_total is None else adaptive_total
    L.check(L.lib().adakv_safeguard_blend(_ptr(a), int(at), int(total), int(h), float(alpha), _ptr(c), _ptr(out)))
    return out[:int(h)]


def repair_zero_budgets(counts, caps):
    c = _i64(counts).copy()
    L.check(L.lib().adakv_repair_zero_budgets(_ptr(c), _ptr(_i64(caps)), c.size))
    return c


def pyramid_layer_budgets(avg, layers, beta_max, beta_min):
    out = np.zeros(max(int(layers), 1), np.int64)
    L.check(L.lib().adakv_pyramid_layer_budgets(int(avg), int(layers), float(beta_max), float(beta_min), _ptr(out)))
    return out[:int(layers)]
