"""Eviction-quality metrics on device outputs.

Restates the reference's theory helpers (eviction_loss.hpp) over the GPU's scores, keep masks
and decode outputs, so the paper's claim -- adaptive allocation retains more attention mass
than uniform allocation at the same budget (Theorem 3.3 / Fig. 3) -- can be checked
at full model scale:
  * l1_eviction_loss(y, y_hat)        = ||y - y_hat||_1                  (eviction_loss.hpp:18-24)
  * retained_mass(weights, keep)      = sum_i sum_j I_i^j A_i^j          (eviction_loss.hpp:64-78)
  * epsilon_bound(weights, keep, C)   = 2 C * evicted mass               (eviction_loss.hpp:44-61)
Weights are the observation-window scores of each KV group (the mean pooled attention the
selection ranks by); sums run in fp64 on the device.
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
