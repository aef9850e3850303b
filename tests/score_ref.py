"""Torch fp64 restatement of the reference's observation-window scoring, for checking the
GPU scores of WHOLE layers (every group of every problem) at full size.  Test
infrastructure only, like oracle/: it is what the tcgen05 scores are compared against,
never a product path.

Follows policies.hpp:119-132 (window_scores: per window row, softmax over the OUTSIDE keys
of q.k * 1/sqrt(d) -- attention.hpp:141-179 -- then maxpool_same with padded cells
excluded, policies.hpp:99-112, then the mean over rows) and policies.hpp:136-156
(group_mean_scores: mean over the g member heads).  Pinned against the C oracle
(oracle/adakv_oracle.c) in tests/test_gpu_score_parity.py on shapes the oracle finishes in
seconds.
"""
import torch
import torch.nn.functional as F


def window_scores_f64(q, k, pool_kernel=7, scale=True):
    """q [H, m, d], k [G, n, d] (the window = last m rows of k is NOT scored); returns the group
    scores [G, n - m] and the per-head scores [H, n - m], fp64, on q's device."""
    H, m, d = q.shape
    G, n, _ = k.shape
    n_o = n - m
    g = H // G
    q64 = q.to(torch.float64)
    out_h = torch.empty((H, n_o), dtype=torch.float64, device=q.device)
    inv = 1.0 / (d ** 0.5) if scale else 1.0
    pad = (pool_kernel - 1) // 2
    for gi in range(G):
        kg = k[gi, :n_o].to(torch.float64)
        for h in range(gi * g, (gi + 1) * g):
            logits = (q64[h] @ kg.T) * inv                      # [m, n_o]
            a = torch.softmax(logits, dim=1)                    # max-subtracted, exact fp64
            # stride 1, symmetric pad, padded cells excluded (max_pool1d pads with -inf)
            pooled = F.max_pool1d(a[None], pool_kernel, stride=1, padding=pad)[0] if pad else a
            out_h[h] = pooled.sum(dim=0) / m
    out_g = out_h.view(G, g, n_o).sum(dim=1) / g
    return out_g, out_h
