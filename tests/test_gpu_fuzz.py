"""Seeded random sweep of the whole path on the device: random shapes (problems, KV groups,
group sizes 1-8, window, prompt, head dim 64/128), pool kernels, kinds and budgets, through
adakv_compress (tcgen05 scoring where the shape allows it, the SIMT kernels otherwise) and
one decode step with its append.  Per case:
  * the oracle's selection (budget.hpp:118-158, policies.hpp:80-93, 178-196) fed the device's
    own scores reproduces budgets and keep masks bit-exactly, and the cache holds exactly the
    kept rows then the window rows of every group (policies.hpp:273-290);
  * the decode output is within the bf16 tolerance of the fp64 attention over those rows plus
    the appended one (attention.hpp:169-196), and the appended row lands at the segment end.
48 cases by default (ADAKV_FUZZ_CASES: 300 measured green).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402


def _case(seed):
    rng = np.random.default_rng(seed)
    P = int(rng.integers(1, 4))
    G = int(rng.choice([1, 2, 3, 4, 5, 8, 13]))
    g = int(rng.choice([1, 2, 3, 4, 6, 8]))
    m = int(rng.choice([4, 8, 32, 32]))
    d = int(rng.choice([64, 128, 128]))
    n_o = int(rng.integers(m + 1, 1200))
    pool = int(rng.choice([1, 3, 5, 7]))
    kind = str(rng.choice(["ada_snapkv", "ada_snapkv", "snapkv"]))
    lb = int(rng.integers(m * G + G, G * (n_o + m) + 1))
    return P, G, g, m, d, n_o, pool, kind, lb


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADAKV_FUZZ_CASES", "48"))))
def test_random_compress_then_decode(dev, oracle_mod, seed):
    O = oracle_mod
    P, G, g, m, d, n_o, pool, kind, lb = _case(seed)
    H = G * g
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=100 + seed, dtype=torch.bfloat16, device=dev)
    c = A.compress(q, k, v, lb, kind=kind, pool_kernel=pool, alpha=0.2, reserve=2, return_scores=True,
                   return_keep=True, check=True)
    outside = lb - m * G
    kk, vv = k.cpu(), v.cpu()
    for p in range(P):
        s64 = c.scores[p].double().cpu().numpy()
        caps = np.full(G, n_o)
        if kind == "ada_snapkv":
            raw = O.adaptive_allocation(list(s64), outside)
            b = O.repair_zero_budgets(O.safeguard_blend(raw, outside, G, 0.2, caps), caps)
        else:
            b = O.repair_zero_budgets(O.uniform_allocation(outside, G, caps), caps)
        keep = np.stack([O.topk_decision(s64[i], int(b[i])) for i in range(G)])
        assert c.budgets[p * G:(p + 1) * G].cpu().tolist() == b.tolist(), (seed, p)
        assert np.array_equal(c.keep[p].cpu().numpy(), keep), (seed, p)
        for i in range(G):
            idx = np.concatenate([np.nonzero(keep[i])[0], n_o + np.arange(m)])
            kr, vr = c.segment(p, i)
            assert torch.equal(kr.cpu().view(torch.int16), kk[p, i, idx].view(torch.int16)), (seed, p, i)
            assert torch.equal(vr.cpu().view(torch.int16), vv[p, i, idx].view(torch.int16)), (seed, p, i)
    # one decode step with its append, against fp64 attention over the retained rows + the new one
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    qd = torch.randn((P, H, d), generator=gen, device=dev).to(torch.bfloat16)
    kn = torch.randn((P, G, d), generator=gen, device=dev).to(torch.bfloat16)
    vn = torch.randn((P, G, d), generator=gen, device=dev).to(torch.bfloat16)
    before = c.seqlens.clone()
    o = A.decode(qd, c, kn, vn, check=True)
    assert torch.equal(c.seqlens, before + 1)
    for p in range(P):
        for i in range(G):
            kr, vr = c.segment(p, i)
            assert torch.equal(kr[-1].view(torch.int16), kn[p, i].view(torch.int16))
            assert torch.equal(vr[-1].view(torch.int16), vn[p, i].view(torch.int16))
            kr64, vr64 = kr.double(), vr.double()
            for h in range(i * g, (i + 1) * g):
                w = torch.softmax(kr64 @ qd[p, h].double() / d ** 0.5, dim=0)
                ref = w @ vr64
                err = (o[p, h].double() - ref).abs().max().item()
                assert err <= 2e-2 and err <= 1e-2 * max(ref.abs().max().item(), 1e-3) + 4e-3, (seed, p, h, err)


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADAKV_FUZZ_SELECT_CASES", "24"))))
def test_random_segmented_select(dev, oracle_mod, seed):
    """Random selection problems straight through adakv_segmented_select: 1-40 problems, 1-64
    ragged non-empty segments (the lean layout past 39), up to ~600K keys per problem (clusters
    of up to 16 CTAs, slices streamed from L2), heavy ties, f32 or f64 keys, adaptive (blended,
    repaired) or uniform allocation -- budgets and keep masks bit-exact to evict_rows
    (policies.hpp:298-323), kept positions in flat order."""
    O = oracle_mod
    rng = np.random.default_rng(1000 + seed)
    P = int(rng.integers(1, 41)) if seed % 3 else 1
    S = int(rng.choice([1, 2, 5, 8, 16, 39, 40, 64]))
    big = seed % 4 == 0
    sizes = rng.integers(1, (600000 // S) if big else 3000, size=S)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    N = int(off[-1])
    levels = int(rng.choice([8, 64, 4096]))
    x = np.floor(rng.random((P, N)) * levels) / levels
    dt = torch.float64 if seed % 5 == 0 else torch.float32
    s = torch.as_tensor(x, dtype=dt, device=dev)
    adaptive = bool(seed % 2 == 0)
    total = int(rng.integers(S, N + 1))
    r = A.segmented_select(s, off, total, "adaptive" if adaptive else "uniform", blend=adaptive, alpha=0.2,
                           repair=True)
    for p in range(min(P, 3)):
        rows = [x[p, off[i]:off[i + 1]] for i in range(S)]
        alloc, keep = O.evict_rows(rows, total, adaptive, 0.2)
        assert r["budgets"][p].cpu().tolist() == alloc.tolist(), (seed, p)
        kp = np.concatenate(keep)
        assert np.array_equal(r["keep"][p].cpu().numpy(), kp), (seed, p)
        pos = np.concatenate([np.nonzero(k)[0] for k in keep])
        assert np.array_equal(r["kept_pos"][p, :total].cpu().numpy(), pos), (seed, p)
    A.workspace_status(r["ws"])


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADAKV_FUZZ_GENERIC_CASES", "16"))))
def test_random_generic_dtypes_and_kinds(dev, oracle_mod, seed):
    """The SIMT paths: f32 / f64 layers (scores from the generic kernels, decode on the generic
    split-K kernel), every kind including StreamingLLM and per-problem (pyramid) budgets,
    optionally with V in pinned host memory -- selection bit-exact on the device's own scores,
    retained rows exact, decode within fp32 / fp64 tolerance of fp64 attention."""
    O = oracle_mod
    rng = np.random.default_rng(5000 + seed)
    dt = torch.float64 if seed % 2 else torch.float32
    P = int(rng.integers(1, 4))
    G = int(rng.choice([1, 2, 3, 4, 8]))
    g = int(rng.choice([1, 2, 4]))
    m = int(rng.choice([2, 8, 16]))
    d = int(rng.choice([16, 64, 128]))
    n_o = int(rng.integers(m + 1, 700))
    pool = int(rng.choice([1, 3, 5, 7, 9]))
    kind = str(rng.choice(["ada_snapkv", "snapkv", "streaming_llm", "ada_pyramid"]))
    H = G * g
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=200 + seed, dtype=dt, device=dev)
    lb_per = rng.integers(m * G + G, G * (n_o + m) + 1, size=P)
    per_problem = kind == "ada_pyramid"
    lb = int(lb_per[0])
    vin = v.cpu().pin_memory() if seed % 3 == 0 else v
    c = A.compress(q, k, vin, lb, kind=kind, pool_kernel=pool, alpha=0.2, reserve=1, return_scores=True,
                   return_keep=True, check=True,
                   layer_budgets=torch.as_tensor(lb_per, device=dev) if per_problem else None)
    kk, vv = k.cpu(), v.cpu()
    for p in range(P):
        outside = int(lb_per[p] if per_problem else lb) - m * G
        s64 = c.scores[p].double().cpu().numpy()
        caps = np.full(G, n_o)
        if kind in ("ada_snapkv", "ada_pyramid"):
            raw = O.adaptive_allocation(list(s64), outside)
            b = O.repair_zero_budgets(O.safeguard_blend(raw, outside, G, 0.2, caps), caps)
        else:
            b = O.repair_zero_budgets(O.uniform_allocation(outside, G, caps), caps)
        if kind == "streaming_llm":
            keep = np.stack([O.streaming_llm_decision(n_o, min(4, int(x)), int(x) - min(4, int(x))) for x in b])
        else:
            keep = np.stack([O.topk_decision(s64[i], int(b[i])) for i in range(G)])
        assert c.budgets[p * G:(p + 1) * G].cpu().tolist() == b.tolist(), (seed, p)
        assert np.array_equal(c.keep[p].cpu().numpy(), keep), (seed, p)
        for i in range(G):
            idx = np.concatenate([np.nonzero(keep[i])[0], n_o + np.arange(m)])
            kr, vr = c.segment(p, i)
            assert torch.equal(kr.cpu(), kk[p, i, idx]) and torch.equal(vr.cpu(), vv[p, i, idx]), (seed, p, i)
    qd = torch.as_tensor(rng.normal(size=(P, H, d)), dtype=dt, device=dev)
    kn = torch.as_tensor(rng.normal(size=(P, G, d)), dtype=dt, device=dev)
    vn = torch.as_tensor(rng.normal(size=(P, G, d)), dtype=dt, device=dev)
    o = A.decode(qd, c, kn, vn, check=True)
    tol = 1e-10 if dt == torch.float64 else 2e-5
    for p in range(P):
        for i in range(G):
            kr, vr = c.segment(p, i)
            for h in range(i * g, (i + 1) * g):
                w = torch.softmax(kr.double() @ qd[p, h].double() / d ** 0.5, dim=0)
                ref = w @ vr.double()
                err = (o[p, h].double() - ref).abs().max().item()
                assert err <= tol * max(1.0, ref.abs().max().item()), (seed, p, h, err)


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADAKV_FUZZ_SHARD_CASES", "12"))))
def test_random_kv_group_sharded_compress_matches_compress(dev, seed):
    """The KV-group-sharded compress (local top-k, the device-packed payload, the candidate union,
    the merged allocation, the per-group selection; world size 1) equals the single-GPU compress
    on random shapes: budgets, segment lengths and every retained row bit for bit."""
    from paper_2407_11550_b200.sharding import compress_kv_group_sharded
    rng = np.random.default_rng(7000 + seed)
    G = int(rng.choice([1, 2, 4, 8]))
    g = int(rng.choice([1, 2, 4, 8]))
    m, d = 32, 128
    n_o = int(rng.integers(64, 3000))
    H = G * g
    q, k, v = planted_layer(1, H, G, n_o, m, d, seed=300 + seed, dtype=torch.bfloat16, device=dev)
    lb = int(rng.integers(m * G + G, G * (n_o + m) + 1))
    ref = A.compress(q, k, v, lb, reserve=2)
    sh, _ = compress_kv_group_sharded(q[0], k[0], v[0], lb, G, g0=0, reserve=2)
    assert torch.equal(sh.budgets.cpu(), ref.budgets.cpu()), seed
    assert torch.equal(sh.seqlens.cpu(), ref.seqlens.cpu()), seed
    for i in range(G):
        kr, vr = ref.segment(0, i)
        ks, vs = sh.segment(0, i)
        assert torch.equal(ks.view(torch.int16), kr.view(torch.int16)), (seed, i)
        assert torch.equal(vs.view(torch.int16), vr.view(torch.int16)), (seed, i)
