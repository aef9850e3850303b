"""Full-size GPU checks at the BASELINE.json configurations that are not bench lines
(configs 3, 4 and 5), through size-independent properties.

For every problem of a compressed layer:
  * budgets: the oracle's adaptive_allocation + safeguard_blend + repair (budget.hpp:118-158,
    policies.hpp:178-196) fed the GPU's own scores gives the GPU's budgets BIT-EXACTLY, and they
    sum to layer_budget - m*G;
  * decisions: the oracle's topk_decision (policies.hpp:80-93) on the same scores equals the
    GPU keep mask;
  * compaction: every segment is exactly k[p, g, kept positions] followed by the m window rows
    (policies.hpp:273-290), bit for bit;
  * scores: one group against the fp64 oracle on the same bf16 values, |d| <= 1e-4 * max;
  * decode: one step over the compacted cache against the fp64 oracle, bf16 tolerance.
Config 3 also exercises the select kernel's global-memory path (1M scores per problem do not
fit a cluster's shared memory) and config 4 the generic scoring kernel (g*m = 256 rows).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200.sharding import CudaSelector, kv_group_sharded_allocation  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402


def _check_layer(O, q, k, v, cache, LB, alpha=0.2, score_group=None, decode_problems=(0,)):
    P, H, m, d = q.shape
    G, n = k.shape[1], k.shape[2]
    n_o = n - m
    gs = H // G
    outside = LB - m * G
    budgets = cache.budgets.view(P, G).cpu().numpy()
    for p in range(P):
        s64 = cache.scores[p].double().cpu().numpy()
        raw = O.adaptive_allocation(list(s64), outside)
        b = O.repair_zero_budgets(O.safeguard_blend(raw, outside, G, alpha, np.full(G, n_o)), np.full(G, n_o))
        assert budgets[p].tolist() == b.tolist(), p
        assert int(budgets[p].sum()) == outside
        keep = cache.keep[p].cpu().numpy()
        for g in range(G):
            assert np.array_equal(keep[g], O.topk_decision(s64[g], int(b[g]))), (p, g)
            pos = torch.as_tensor(np.concatenate([np.nonzero(keep[g])[0], n_o + np.arange(m)]), device=k.device)
            kr, vr = cache.segment(p, g)
            assert torch.equal(kr, k[p, g].index_select(0, pos)) and torch.equal(vr, v[p, g].index_select(0, pos))
    if score_group is not None:
        p, g = score_group
        q64 = q[p].double().cpu().numpy()
        k64 = k[p, g, :n_o].double().cpu().numpy()
        per = [O.window_scores(q64[h], k64, 7) for h in range(g * gs, (g + 1) * gs)]
        ref = O.group_mean_scores(np.stack(per), gs)[0]
        assert np.abs(cache.scores[p, g].double().cpu().numpy() - ref).max() <= 1e-4 * ref.max()
    gen = torch.Generator(device=q.device)
    gen.manual_seed(1)
    qd = torch.randn((P, H, d), generator=gen, device=q.device).to(q.dtype)
    o = A.decode(qd, cache)
    for p in decode_problems:
        segs = [cache.segment(p, g) for g in range(G)]
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd[p].double().cpu().numpy(), torch.cat([s[0] for s in segs]).double().cpu().numpy(),
                                 torch.cat([s[1] for s in segs]).double().cpu().numpy(), off)
        err = np.abs(o[p].double().cpu().numpy() - ref).max()
        assert err <= 2e-2 and err <= 1e-2 * max(np.abs(ref).max(), 1e-3) + 4e-3, (p, err)


@pytest.mark.parametrize("budget", [128, 1024, 4096])
def test_config3_mistral_128k_batch8(dev, oracle_mod, budget):
    """Config 3: Mistral-7B shapes (32 Q / 8 KV heads), 128K prompt, batch 8, budget sweep."""
    P, H, G, m, d, n = 8, 32, 8, 32, 128, 131072
    q, k, v = planted_layer(P, H, G, n - m, m, d, seed=30 + budget, dtype=torch.bfloat16, device=dev)
    LB = budget * G
    cache = A.compress(q, k, v, LB, kind="ada_snapkv", pool_kernel=7, alpha=0.2, reserve=2, return_scores=True,
                       return_keep=True)
    _check_layer(oracle_mod, q, k, v, cache, LB, score_group=(3, 5) if budget == 1024 else None,
                 decode_problems=(0, 7))


def test_config4_llama70b_64k_group_sharded_merge(dev, oracle_mod):
    """Config 4: Llama-3.1-70B shapes (64 Q / 8 KV heads, g = 8), 64K prompt, budget 2048.
    The whole layer on one GPU, plus the KV-group-sharded allocation (one all-gather of top-k
    candidates, sharding.py) at world size 1 reproducing the single-GPU budgets and decisions."""
    P, H, G, m, d, n = 1, 64, 8, 32, 128, 65536
    q, k, v = planted_layer(P, H, G, n - m, m, d, seed=41, dtype=torch.bfloat16, device=dev)
    LB = 2048 * G
    cache = A.compress(q, k, v, LB, kind="ada_snapkv", pool_kernel=7, alpha=0.2, reserve=2, return_scores=True,
                       return_keep=True)
    _check_layer(oracle_mod, q, k, v, cache, LB, score_group=(0, 2))
    r = kv_group_sharded_allocation(cache.scores[0], 0, G, LB - m * G, 0.2, CudaSelector())
    assert r.budgets.tolist() == cache.budgets.cpu().tolist()
    keep = cache.keep[0].cpu().numpy()
    kept = r.kept(0, G)
    for g in range(G):
        assert kept[g].tolist() == np.nonzero(keep[g])[0].tolist()


def test_config5_question_agnostic_batch4(dev, oracle_mod):
    """Config 5: Llama-3.1-8B shapes, 32K context, budget 1024/head, 4 requests per GPU (32 on
    8 GPUs).  The window is the last 32 context tokens (question-agnostic); the kernels are the
    same, only the caller's choice of window differs."""
    P, H, G, m, d, n = 4, 32, 8, 32, 128, 32768
    q, k, v = planted_layer(P, H, G, n - m, m, d, seed=52, dtype=torch.bfloat16, device=dev)
    LB = 1024 * G
    cache = A.compress(q, k, v, LB, kind="ada_snapkv", pool_kernel=7, alpha=0.2, reserve=2, return_scores=True,
                       return_keep=True)
    _check_layer(oracle_mod, q, k, v, cache, LB, score_group=(2, 7), decode_problems=(0, 3))
