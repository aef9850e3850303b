"""Eviction-quality evaluation on device outputs.

Restates the reference's theory helpers (eviction_loss.hpp) and its policy comparison
(report.hpp:161-345) over the GPU's scores, budgets, keep masks and decode outputs, so the
paper's claim -- adaptive allocation beats uniform allocation at the same budget (PAPER.md
Theorem 3.3 / Fig. 3; acceptance_test.cpp:134-163) -- is checked on what the CUDA path produces:
  * l1_eviction_loss(y, y_hat)        = ||y - y_hat||_1                  (eviction_loss.hpp:18-24)
  * row_norm_constant(V, W_o)         = max_i max_r ||(V_i W_i^O)_r||_1  (eviction_loss.hpp:26-41)
  * epsilon_bound(weights, keep, C)   = 2 C * evicted mass               (eviction_loss.hpp:44-61)
  * retained_mass(weights, keep)      = sum_i sum_j I_i^j A_i^j          (eviction_loss.hpp:64-78)
  * epsilon_star(w, budgets, C)       = 2 C (h - sum_i topk-mass_i)      (eviction_loss.hpp:97-109)
  * epsilon_double_star(w, B, C)      = 2 C (h - global top-B mass)      (eviction_loss.hpp:111-127)
  * comparison_rows / run_comparison  = report.hpp:216-249 + 322-345 for a full trace: the
    loss of the GPU's compressed cache (decoded by the GPU kernel) against full attention,
    the bound ladder against the decode query's true weights, and the win fraction.
Sums run in fp64 on the device.
"""
from __future__ import annotations

import torch

from . import _lib as L


def l1_eviction_loss(y: torch.Tensor, y_hat: torch.Tensor) -> float:
    if y.shape != y_hat.shape:
        raise L.InvalidArgument(1, "l1_eviction_loss: length mismatch")
    return float((y.double() - y_hat.double()).abs().sum())


def retained_mass(weights: torch.Tensor, keep: torch.Tensor) -> torch.Tensor:
    """weights [..., n], keep [..., n] (0/1) -> retained mass summed over the last two dims
    (heads/groups and positions) for every leading index."""
    if weights.shape != keep.shape:
        raise L.InvalidArgument(1, "retained_mass: decision length mismatch")
    return (weights.double() * (keep != 0)).sum(dim=(-2, -1))


def epsilon_bound(weights: torch.Tensor, keep: torch.Tensor, c: float) -> torch.Tensor:
    if weights.shape != keep.shape:
        raise L.InvalidArgument(1, "epsilon_bound: decision length mismatch")
    if c < 0:
        raise L.InvalidArgument(1, "epsilon_bound: negative constant")
    return 2.0 * c * (weights.double() * (keep == 0)).sum(dim=(-2, -1))


def compare_allocations(q, k, v, layer_budget, alpha=0.2, pool_kernel=7):
    """Ada-KV (ada_snapkv) against uniform allocation (snapkv) on the same layers: the retained
    window-score mass per problem for each, and the L1 distance of one decode step (the last
    window query of every head) from full-cache attention.  Returns a dict of per-problem
    tensors."""
    from . import ops
    P, H, m, d = q.shape
    G, n = k.shape[1], k.shape[2]
    ada = ops.compress(q, k, v, layer_budget, kind="ada_snapkv", alpha=alpha, pool_kernel=pool_kernel,
                       return_scores=True, return_keep=True)
    uni = ops.compress(q, k, v, layer_budget, kind="snapkv", pool_kernel=pool_kernel, return_scores=True,
                       return_keep=True)
    res = {"retained_ada": retained_mass(ada.scores, ada.keep), "retained_uniform": retained_mass(uni.scores, uni.keep)}
    # one decode step: query = the last window row of every head; full attention as reference
    qd = q[:, :, m - 1, :].contiguous()
    o_ada, o_uni = ops.decode(qd, ada), ops.decode(qd, uni)
    qg = qd.double().view(P, G, H // G, d)
    att = torch.softmax(torch.einsum("pgsd,pgnd->pgsn", qg, k.double()) / d ** 0.5, dim=-1)
    full = torch.einsum("pgsn,pgnd->pgsd", att, v.double()).reshape(P, H, d)
    res["l1_ada"] = (o_ada.double() - full).abs().sum(dim=(1, 2))
    res["l1_uniform"] = (o_uni.double() - full).abs().sum(dim=(1, 2))
    return res


def row_norm_constant(v: torch.Tensor, wo: torch.Tensor) -> float:
    """v [h, n, d] (each head's full value rows), wo [h, d, D] -> C (eviction_loss.hpp:26-41)."""
    if v.shape[0] == 0:
        raise L.InvalidArgument(1, "row_norm_constant: empty cache")
    if v.shape[0] != wo.shape[0]:
        raise L.InvalidArgument(1, "row_norm_constant: head count mismatch")
    return float(torch.einsum("hnd,hdD->hnD", v.double(), wo.double()).abs().sum(dim=-1).max())


def _topk_mass(w: torch.Tensor, k: torch.Tensor) -> torch.Tensor:
    """sum of the k[i] largest entries of every row of w [r, n] (k int tensor [r])."""
    srt = torch.sort(w.double(), dim=-1, descending=True).values
    idx = torch.arange(w.shape[-1], device=w.device)[None, :]
    return (srt * (idx < k[:, None].to(w.device))).sum(dim=-1)


def epsilon_star(weights: torch.Tensor, budgets: torch.Tensor, c: float) -> torch.Tensor:
    """weights [..., h, n], budgets [..., h] -> 2 C (h - sum_i topk-mass_i) per leading index."""
    lead = weights.shape[:-2]
    h, n = weights.shape[-2:]
    km = _topk_mass(weights.reshape(-1, n), budgets.reshape(-1)).reshape(*lead, h)
    return 2.0 * c * (h - km.sum(dim=-1))


def epsilon_double_star(weights: torch.Tensor, total, c: float) -> torch.Tensor:
    """weights [..., h, n], total (int or tensor [...]) -> 2 C (h - mass of the global top-total)."""
    lead = weights.shape[:-2]
    h, n = weights.shape[-2:]
    flat = weights.reshape(-1, h * n)
    t = torch.as_tensor(total, device=weights.device).reshape(-1).expand(flat.shape[0])
    return 2.0 * c * (h - _topk_mass(flat, t).reshape(lead))


def comparison_rows(q_win, k_out, v_out, k_win, v_win, q_dec, wo, layer_budget, kind="ada_snapkv", alpha=0.2,
                    pool_kernel=7):
    """report.hpp:216-249 for P samples at once (a full trace, one layer): the device compress
    (evict_layer) decides, the device decode over the compressed cache gives y_hat (a fresh
    softmax over the retained rows, output_from_retained), and the bound ladder is evaluated
    against the decode query's true weights over the full cache.
    q_win [P, H, m, d], k_out/v_out [P, G, n, d], k_win/v_win [P, G, m, d], q_dec [P, H, d],
    wo [H, d, D] (same dtype; fp64 runs the device's fp64 path).  Returns per-sample tensors:
    loss, epsilon, epsilon_star, epsilon_double_star, mass, alloc [P, G]."""
    from . import ops
    P, H, m, d = q_win.shape
    G, n = k_out.shape[1], k_out.shape[2]
    g = H // G
    k = torch.cat([k_out, k_win], dim=2).contiguous()
    v = torch.cat([v_out, v_win], dim=2).contiguous()
    cache = ops.compress(q_win.contiguous(), k, v, layer_budget, kind=kind, alpha=alpha, pool_kernel=pool_kernel,
                         return_scores=True, return_keep=True, check=True)
    o = ops.decode(q_dec.contiguous(), cache)                                  # [P, H, d]
    wo64 = wo.double()
    y_hat = torch.einsum("phd,hdD->pD", o.double(), wo64)
    # true weights of the decode query over each head's full cache (outside, then window)
    kh = k.double().repeat_interleave(g, dim=1)                                # [P, H, n + m, d]
    vh = v.double().repeat_interleave(g, dim=1)
    w = torch.softmax(torch.einsum("phd,phnd->phn", q_dec.double(), kh) / d ** 0.5, dim=-1)
    y = torch.einsum("phn,phnd,hdD->pD", w, vh, wo64)
    c = torch.einsum("phnd,hdD->phnD", vh, wo64).abs().sum(dim=-1).amax(dim=(1, 2))  # [P]
    keep = torch.cat([cache.keep.repeat_interleave(g, dim=1),
                      torch.ones((P, H, m), dtype=cache.keep.dtype, device=k.device)], dim=2)
    evicted = (w * (keep == 0)).sum(dim=(1, 2))
    mass = (w * (keep != 0)).sum(dim=(1, 2))
    bud = cache.budgets.view(P, G)
    scores = cache.scores.double()
    return {"loss": (y - y_hat).abs().sum(dim=1), "epsilon": 2.0 * c * evicted,
            "epsilon_star": epsilon_star(scores, bud, 1.0),
            "epsilon_double_star": epsilon_double_star(scores, bud.sum(dim=1), 1.0), "mass": mass, "alloc": bud}


def run_comparison(q_win, k_out, v_out, k_win, v_win, q_dec, wo, fractions=(0.2, 0.4), alpha=0.2, pool_kernel=7,
                   policies=("ada_snapkv", "snapkv")):
    """The policy comparison of report.hpp:161-345 over P samples of one full-trace layer:
    layer budget = ceil(fraction * G (n + m)) (capped), every policy's rows, and the fraction of
    samples on which the adaptive policy's loss is strictly below the baseline's."""
    import math
    P, G, n, _ = k_out.shape
    m = k_win.shape[2]
    unique = G * (n + m)
    rows, aggregates = {}, {}
    for f in fractions:
        lb = min(int(math.ceil(f * unique)), unique)
        for pol in policies:
            rows[(f, pol)] = comparison_rows(q_win, k_out, v_out, k_win, v_win, q_dec, wo, lb, kind=pol, alpha=alpha,
                                             pool_kernel=pool_kernel)
        if "ada_snapkv" in policies and "snapkv" in policies:
            wins = (rows[(f, "ada_snapkv")]["loss"] < rows[(f, "snapkv")]["loss"]).sum()
            aggregates[f] = float(wins) / P
    return rows, aggregates
