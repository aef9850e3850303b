"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/liboracle.so`` (the plain-C restatement, adakv_oracle.c) and,
when present, ``oracle/_ref/libadakv_ref.so`` (the reference's own headers
compiled in place by ``make ref``).  Both expose the same calling convention,
so every helper below takes ``impl="oracle"`` or ``impl="ref"``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libadakv_ref.so")

I64 = C.c_int64
DBL = C.c_double
PD = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
PI = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
PU8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")

KINDS = {"snapkv": 0, "pyramid": 1, "ada_snapkv": 2, "ada_pyramid": 3, "streaming_llm": 4}


class OracleError(Exception):
    """Mirror of the reference's exception channel (status 1/2/3)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status
        self.kind = {1: "invalid_argument", 2: "out_of_range"}.get(status, "error")


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_libs: dict[str, C.CDLL] = {}


def _opt_ptr(arr, typ):
    return None if arr is None else arr.ctypes.data_as(C.POINTER(typ))


def lib(impl: str = "oracle") -> C.CDLL:
    if impl in _libs:
        return _libs[impl]
    if impl == "oracle":
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        L.orc_last_error.restype = C.c_char_p
        prefix = "orc_"
    elif impl == "ref":
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        prefix = "ref_"
    else:
        raise ValueError(impl)
    L._prefix = prefix
    _libs[impl] = L
    return L


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _call(impl: str, name: str, *args):
    L = lib(impl)
    fn = getattr(L, L._prefix + name)
    fn.restype = C.c_int
    st = fn(*args)
    if st != 0:
        msg = getattr(L, L._prefix + "last_error")().decode()
        raise OracleError(st, msg)


def _d(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _i(x):
    return np.ascontiguousarray(x, dtype=np.int64)


def topk_decision(a, k, impl="oracle"):
    a = _d(a)
    keep = np.zeros(a.size, np.uint8)
    _call(impl, "topk_decision", a.ctypes.data_as(C.POINTER(DBL)), I64(a.size), I64(k),
          keep.ctypes.data_as(C.POINTER(C.c_uint8)))
    return keep


def attention_weights(q, keys, scale=True, impl="oracle"):
    q, keys = _d(np.atleast_2d(q)), _d(keys)
    m, d = q.shape
    n = keys.shape[0]
    out = np.zeros((m, n))
    _call(impl, "attention_weights", q.ctypes.data_as(C.POINTER(DBL)), I64(m),
          keys.ctypes.data_as(C.POINTER(DBL)), I64(n), I64(d), C.c_int(int(scale)),
          out.ctypes.data_as(C.POINTER(DBL)))
    return out


def window_scores(q, keys, pool_kernel, scale=True, impl="oracle"):
    q, keys = _d(np.atleast_2d(q)), _d(keys)
    m, d = q.shape
    n = keys.shape[0]
    out = np.zeros(n)
    _call(impl, "window_scores", q.ctypes.data_as(C.POINTER(DBL)), I64(m),
          keys.ctypes.data_as(C.POINTER(DBL)), I64(n), I64(d), I64(pool_kernel),
          C.c_int(int(scale)), out.ctypes.data_as(C.POINTER(DBL)))
    return out


def group_mean_scores(scores, g, impl="oracle"):
    s = _d(scores)
    h, n = s.shape
    out = np.zeros((max(h // g, 0) if g else 0, n))
    _call(impl, "group_mean_scores", s.ctypes.data_as(C.POINTER(DBL)), I64(h), I64(n), I64(g),
          out.ctypes.data_as(C.POINTER(DBL)))
    return out


def apportion(quotas, total, caps=None, impl="oracle"):
    q = _d(quotas)
    out = np.zeros(q.size, np.int64)
    c = None if caps is None else _i(caps)
    _call(impl, "apportion", q.ctypes.data_as(C.POINTER(DBL)), I64(q.size), I64(total),
          _opt_ptr(c, I64), out.ctypes.data_as(C.POINTER(I64)))
    return out


def uniform_allocation(total, h, caps=None, impl="oracle"):
    out = np.zeros(h, np.int64)
    c = None if caps is None else _i(caps)
    _call(impl, "uniform_allocation", I64(total), I64(h), _opt_ptr(c, I64),
          out.ctypes.data_as(C.POINTER(I64)))
    return out


def _ragged(rows):
    rows = [np.asarray(r, np.float64).ravel() for r in rows]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([r.size for r in rows])
    flat = np.concatenate(rows) if rows else np.zeros(0)
    return _d(flat), off


def adaptive_allocation(rows, total, impl="oracle"):
    flat, off = _ragged(rows)
    h = len(rows)
    out = np.zeros(h, np.int64)
    _call(impl, "adaptive_allocation", flat.ctypes.data_as(C.POINTER(DBL)),
          off.ctypes.data_as(C.POINTER(I64)), I64(h), I64(total), out.ctypes.data_as(C.POINTER(I64)))
    return out


def safeguard_blend(adaptive, total, h, alpha, caps=None, adaptive_total=None, impl="oracle"):
    a = _i(adaptive)
    out = np.zeros(h, np.int64)
    c = None if caps is None else _i(caps)
    at = total if adaptive_total is None else adaptive_total
    _call(impl, "safeguard_blend", a.ctypes.data_as(C.POINTER(I64)), I64(at), I64(total), I64(h),
          DBL(alpha), _opt_ptr(c, I64), out.ctypes.data_as(C.POINTER(I64)))
    return out


def pyramid_layer_budgets(avg, layers, beta_max, beta_min, impl="oracle"):
    out = np.zeros(max(layers, 1), np.int64)
    _call(impl, "pyramid_layer_budgets", I64(avg), I64(layers), DBL(beta_max), DBL(beta_min),
          out.ctypes.data_as(C.POINTER(I64)))
    return out[:layers]


def repair_zero_budgets(counts, caps, impl="oracle"):
    c = _i(counts).copy()
    cp = _i(caps)
    _call(impl, "repair_zero_budgets", c.ctypes.data_as(C.POINTER(I64)),
          cp.ctypes.data_as(C.POINTER(I64)), I64(c.size))
    return c


def streaming_llm_decision(n, sink, recent, impl="oracle"):
    keep = np.zeros(max(n, 1), np.uint8)
    _call(impl, "streaming_llm_decision", I64(n), I64(sink), I64(recent),
          keep.ctypes.data_as(C.POINTER(C.c_uint8)))
    return keep[:n]


def evict_rows(rows, total, adaptive, alpha=1.0, impl="oracle"):
    flat, off = _ragged(rows)
    h = len(rows)
    alloc = np.zeros(max(h, 1), np.int64)
    keep = np.zeros(max(flat.size, 1), np.uint8)
    _call(impl, "evict_rows", flat.ctypes.data_as(C.POINTER(DBL)),
          off.ctypes.data_as(C.POINTER(I64)), I64(h), I64(total), C.c_int(int(adaptive)),
          DBL(alpha), alloc.ctypes.data_as(C.POINTER(I64)), keep.ctypes.data_as(C.POINTER(C.c_uint8)))
    return alloc[:h], [keep[off[i]:off[i + 1]].copy() for i in range(h)]


@dataclass
class EvictResult:
    group_scores: np.ndarray   # [sum n_g]  (flat; per group rows [off[g], off[g+1]))
    alloc: np.ndarray          # [G]
    keep: np.ndarray           # [sum n_g] uint8
    k_ret: np.ndarray          # [layer_budget, d]
    v_ret: np.ndarray          # [layer_budget, d]
    ret_len: np.ndarray        # [G]
    off: np.ndarray            # [G+1]
    head_scores: np.ndarray | None = None


class _Cfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("window_size", I64), ("pool_kernel", I64), ("alpha", DBL),
                ("sink_tokens", I64), ("gqa_group_size", I64), ("scale", C.c_int)]


def evict_layer(q, k_out, v_out, k_win, v_win, layer_budget, kind="ada_snapkv", pool_kernel=7,
                alpha=0.2, sink_tokens=4, scale=True, window_size=None, impl="oracle"):
    """q [H,m,d]; k_out/v_out either [G,n,d] or a list of G arrays [n_g,d]; k_win/v_win [G,m,d]."""
    q = _d(q)
    H, m, d = q.shape
    if isinstance(k_out, (list, tuple)):
        lens = [np.asarray(x).shape[0] for x in k_out]
        ko = _d(np.concatenate([np.asarray(x).reshape(-1, d) for x in k_out]))
        vo = _d(np.concatenate([np.asarray(x).reshape(-1, d) for x in v_out]))
    else:
        G0, n, _ = np.asarray(k_out).shape
        lens = [n] * G0
        ko, vo = _d(np.asarray(k_out).reshape(-1, d)), _d(np.asarray(v_out).reshape(-1, d))
    G = len(lens)
    off = np.zeros(G + 1, np.int64)
    off[1:] = np.cumsum(lens)
    kw, vw = _d(k_win).reshape(G, m, d), _d(v_win).reshape(G, m, d)
    N = int(off[-1])
    gs = np.zeros(max(N, 1))
    hs = np.zeros(max(N * (H // G if G else 1), 1))
    alloc = np.zeros(max(G, 1), np.int64)
    keep = np.zeros(max(N, 1), np.uint8)
    LB = max(int(layer_budget), 1)
    k_ret = np.zeros((LB, d))
    v_ret = np.zeros((LB, d))
    ret_len = np.zeros(max(G, 1), np.int64)
    ws = m if window_size is None else window_size
    P = lambda a, t=DBL: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    if impl == "oracle":
        cfg = _Cfg(KINDS[kind], ws, pool_kernel, alpha, sink_tokens, H // G if G else 1, int(scale))
        _call(impl, "evict_layer", P(q), P(ko), P(vo), P(off, I64), P(kw), P(vw), I64(H), I64(G),
              I64(m), I64(d), I64(layer_budget), C.byref(cfg), P(hs), P(gs), P(alloc, I64),
              P(keep, C.c_uint8), P(k_ret), P(v_ret), P(ret_len, I64))
    else:
        _call(impl, "evict_layer", P(q), P(ko), P(vo), P(off, I64), P(kw), P(vw), I64(H), I64(G),
              I64(m), I64(d), I64(layer_budget), C.c_int(KINDS[kind]), I64(ws), I64(pool_kernel),
              DBL(alpha), I64(sink_tokens), C.c_int(int(scale)), P(gs), P(alloc, I64),
              P(keep, C.c_uint8), P(k_ret), P(v_ret), P(ret_len, I64))
    total = int(ret_len[:G].sum())
    return EvictResult(gs[:N], alloc[:G], keep[:N], k_ret[:total], v_ret[:total], ret_len[:G], off,
                       hs[:N * (H // G)] if impl == "oracle" else None)


def decode_attention(q, k, v, off, scale=True, impl="oracle"):
    """q [H,d]; k/v flat [off[G], d]; returns ctx [H,d]."""
    q, k, v, off = _d(q), _d(k), _d(v), _i(off)
    H, d = q.shape
    G = off.size - 1
    out = np.zeros((H, d))
    P = lambda a, t=DBL: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _call(impl, "decode_attention", P(q), P(k), P(v), P(off, I64), I64(H), I64(G), I64(d),
          C.c_int(int(scale)), P(out))
    return out


def select_and_compact(k_heads, v_heads, keep_heads, impl="oracle"):
    """Reference flat-cache compaction; returns (data, offsets, lengths)."""
    d = np.asarray(k_heads[0]).shape[1] if len(k_heads) else 0
    lens = np.array([np.asarray(x).shape[0] for x in k_heads], np.int64)
    h = lens.size
    k = _d(np.concatenate([np.asarray(x).reshape(-1, d) for x in k_heads]))
    v = _d(np.concatenate([np.asarray(x).reshape(-1, d) for x in v_heads]))
    keep = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint8) for x in keep_heads]))
    P = lambda a, t=DBL: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    out = np.zeros(max(2 * int(keep.sum()) * d, 1))
    oo = np.zeros(max(h, 1), np.int64)
    ol = np.zeros(max(h, 1), np.int64)
    if impl == "oracle":
        data = np.zeros(max(2 * int(lens.sum()) * d, 1))
        offs = np.zeros(max(h, 1), np.int64)
        _call(impl, "flatten", P(k), P(v), P(lens, I64), I64(h), I64(d), P(data), P(offs, I64))
        _call(impl, "select_and_compact", P(data), P(offs, I64), P(lens, I64), I64(h), I64(d),
              P(keep, C.c_uint8), P(out), P(oo, I64), P(ol, I64))
    else:
        _call(impl, "select_and_compact", P(k), P(v), P(lens, I64), I64(h), I64(d),
              P(keep, C.c_uint8), P(out), P(oo, I64), P(ol, I64))
    return out[:2 * int(keep.sum()) * d], oo[:h], ol[:h]


def bench_evict_layer(q, k_out, v_out, k_win, v_win, layer_budget, threads, units, kind="ada_snapkv",
                      pool_kernel=7, alpha=0.2):
    """Times `units` reference evict_layer calls on `threads` workers (impl=ref only)."""
    q = _d(q)
    H, m, d = q.shape
    G, n, _ = k_out.shape
    off = np.arange(G + 1, dtype=np.int64) * n
    ko, vo = _d(k_out).reshape(-1, d), _d(v_out).reshape(-1, d)
    kw, vw = _d(k_win), _d(v_win)
    secs = DBL(0)
    alloc = np.zeros(G, np.int64)
    P = lambda a, t=DBL: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _call("ref", "bench_evict_layer", P(q), P(ko), P(vo), P(off, I64), P(kw), P(vw), I64(H), I64(G),
          I64(m), I64(d), I64(layer_budget), C.c_int(KINDS[kind]), I64(pool_kernel), DBL(alpha),
          C.c_int(threads), C.c_int(units), C.byref(secs), P(alloc, I64))
    return secs.value, alloc


def bench_decode(q, k, v, off, threads, units):
    q, k, v, off = _d(q), _d(k), _d(v), _i(off)
    H, d = q.shape
    G = off.size - 1
    secs = DBL(0)
    P = lambda a, t=DBL: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _call("ref", "bench_decode", P(q), P(k), P(v), P(off, I64), I64(H), I64(G), I64(d),
          C.c_int(threads), C.c_int(units), C.byref(secs))
    return secs.value


# ---------------------------------------------------------------- run_comparison restated
def _softmax_row(logits):
    """masked_softmax_inplace over every entry (attention.hpp:141-157): max-subtracted, summed
    in index order, then divided."""
    mx = np.max(logits)
    e = np.exp(logits - mx)
    return e / np.sum(e)


def comparison_row(q_win, k_out, v_out, k_win, v_win, q_dec, wo, layer_budget, kind="ada_snapkv", alpha=0.2,
                   pool_kernel=7, impl="oracle"):
    """One (sample, fraction, policy) row of run_comparison for a full trace with one layer and
    no GQA (report.hpp:216-249): evict_layer's decision through the C restatement, then the
    eviction-loss ladder of eviction_loss.hpp against the decode query's true weights (the
    last window token's query over the full cache, make_sample_context report.hpp:104-127).
    Shapes: q_win [h,m,d], k_out/v_out [h,n,d], k_win/v_win [h,m,d], q_dec [h,d], wo [h,d,D].
    Returns dict(loss, epsilon, epsilon_star, epsilon_double_star, mass, alloc)."""
    h, n, d = np.asarray(k_out).shape
    m = np.asarray(k_win).shape[1]
    res = evict_layer(q_win, k_out, v_out, k_win, v_win, layer_budget, kind=kind, pool_kernel=pool_kernel,
                      alpha=alpha, impl=impl)
    inv = 1.0 / np.sqrt(d)
    keys = [np.concatenate([k_out[i], k_win[i]]) for i in range(h)]
    vals = [np.concatenate([v_out[i], v_win[i]]) for i in range(h)]
    true_w = [_softmax_row(keys[i] @ q_dec[i] * inv) for i in range(h)]
    # attention_output (attention.hpp:182-196): y = sum_i (w_i V_i) W_i^O
    y = sum((true_w[i] @ vals[i]) @ wo[i] for i in range(h))
    # row_norm_constant (eviction_loss.hpp:26-41) over the full cache
    c = max(np.abs(vals[i] @ wo[i]).sum(axis=1).max() for i in range(h))
    keep = res.keep.reshape(h, n)
    full_keep = [np.concatenate([keep[i], np.ones(m, np.uint8)]) for i in range(h)]
    # y_hat: a fresh softmax over each head's retained rows (output_from_retained, report.hpp:130-141)
    off = np.concatenate([[0], np.cumsum(res.ret_len)])
    y_hat = 0.0
    for i in range(h):
        kr, vr = res.k_ret[off[i]:off[i + 1]], res.v_ret[off[i]:off[i + 1]]
        y_hat = y_hat + (_softmax_row(kr @ q_dec[i] * inv) @ vr) @ wo[i]
    evicted = sum(true_w[i][full_keep[i] == 0].sum() for i in range(h))
    mass = sum(true_w[i][full_keep[i] != 0].sum() for i in range(h))
    scores = res.group_scores.reshape(h, n)
    alloc = np.asarray(res.alloc)
    topk = lambda row, k: np.sort(row)[::-1][:k].sum() if k else 0.0  # noqa: E731
    eps_s = 2.0 * (h - sum(topk(scores[i], int(alloc[i])) for i in range(h)))
    eps_ss = 2.0 * (h - topk(scores.reshape(-1), int(alloc.sum())))
    return {"loss": float(np.abs(y - y_hat).sum()), "epsilon": float(2.0 * c * evicted), "epsilon_star": float(eps_s),
            "epsilon_double_star": float(eps_ss), "mass": float(mass), "alloc": alloc.copy()}
