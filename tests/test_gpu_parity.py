"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Gates (BASELINE.json north_star):
  * budgets, keep masks and kept positions BIT-EXACT when fed identical scores;
  * retained K/V rows are exact copies;
  * scores and decode outputs within stated tolerances:
      fp64 path  : |d| <= 1e-12 * max_j s_gj      (exp() ulps + sum order only)
      fp32 path  : |d| <= 1e-5 * max_j s_gj
      bf16 inputs: scores vs the oracle on the SAME bf16 values upcast to fp64,
                   |d| <= 1e-4 * max_j s_gj on realistic inputs (fp32 accumulation), with a
                   derived worst case of 2^-11 * s for the fp16 staging of the head sum
                   (tests/test_gpu_score_parity.py); decode outputs
                   max-abs <= 2e-2 and <= 1e-2 * max|o| (bf16 output rounding).
"""
import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402


def T(x, dtype, dev):
    return torch.as_tensor(np.ascontiguousarray(x)).to(device=dev, dtype=dtype)


# --------------------------------------------------------------------------- budget helpers
def test_budget_helpers_bit_exact(dev, oracle_mod):
    O = oracle_mod
    assert A.safeguard_blend([9, 1], 10, 2, 0.2).tolist() == [6, 4]          # budget_test.cpp:170-174
    assert A.uniform_allocation(10, 3).tolist() == [4, 3, 3]                  # budget_test.cpp:45-48
    assert A.pyramid_layer_budgets(100, 3, 1.5, 0.5).tolist() == [150, 100, 50]
    assert A.apportion([3.5, 3.5, 3.0], 8, [10, 10, 10]).tolist() == [3, 3, 2]
    rng = np.random.default_rng(1)
    for _ in range(150):
        h = int(rng.integers(1, 9))
        caps = rng.integers(1, 40, size=h)
        total = int(rng.integers(0, caps.sum() + 1))
        assert np.array_equal(A.uniform_allocation(total, h, caps), O.uniform_allocation(total, h, caps))
        counts = rng.integers(0, 30, size=h)
        t = int(counts.sum())
        alpha = float(rng.random())
        assert np.array_equal(A.safeguard_blend(counts, t, h, alpha), O.safeguard_blend(counts, t, h, alpha))
        q = rng.random(h) * 10
        tot = int(rng.integers(0, 40))
        assert np.array_equal(A.apportion(q, tot), O.apportion(q, tot))
        layers = int(rng.integers(1, 33))
        avg = int(rng.integers(1, 4096))
        bmin = 0.1 + 0.9 * float(rng.random())
        bmax = bmin + 2.0 * float(rng.random())
        assert np.array_equal(A.pyramid_layer_budgets(avg, layers, bmax, bmin),
                              O.pyramid_layer_budgets(avg, layers, bmax, bmin))
        z = counts.copy()
        z[rng.integers(0, h)] = 0
        if z.sum() >= h:
            assert np.array_equal(A.repair_zero_budgets(z, np.full(h, 100)), O.repair_zero_budgets(z, np.full(h, 100)))
    with pytest.raises(A.InvalidArgument):
        A.uniform_allocation(3, 2, [1, 1])


# --------------------------------------------------------------------------- selection
def _oracle_select(O, s64, total, alpha, blend=True, repair=True):
    G, n = s64.shape
    raw = O.adaptive_allocation(list(s64), total)
    b = O.safeguard_blend(raw, total, G, alpha, np.full(G, n)) if blend else raw
    if repair:
        b = O.repair_zero_budgets(b, np.full(G, n))
    keep = np.stack([O.topk_decision(s64[i], int(b[i])) for i in range(G)])
    return raw, b, keep


def _kept_pos(keep):
    return np.concatenate([np.nonzero(row)[0] for row in keep]).astype(np.int32)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_select_golden_config1(dev, oracle_mod, dtype):
    """Reference generator config 1: identical scores -> identical budgets/decisions."""
    O = oracle_mod
    z = load_golden("config1.npz")
    scores = z["scores"]
    h, gqa, n, d_h, window, seed, LB = z["meta"].tolist()
    G = h // gqa
    outside = LB - window * G
    s = T(scores, dtype, dev).reshape(1, G * n)
    r = A.segmented_select(s, np.arange(G + 1) * n, outside, "adaptive", blend=True, alpha=0.2, repair=True,
                           want_raw=True)
    s64 = s.double().cpu().numpy().reshape(G, n)
    raw, b, keep = _oracle_select(O, s64, outside, 0.2)
    if dtype == torch.float64:
        assert b.tolist() == z["alloc"].tolist() == [837, 837, 1454, 837, 837, 837, 1460, 837]
        assert np.array_equal(keep, z["keep"])
    assert r["raw"][0].cpu().tolist() == raw.tolist()
    assert r["budgets"][0].cpu().tolist() == b.tolist()
    assert np.array_equal(r["keep"][0].cpu().numpy().reshape(G, n), keep)
    assert np.array_equal(r["kept_pos"][0, :outside].cpu().numpy(), _kept_pos(keep))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_select_adversarial_ties(dev, oracle_mod, dtype):
    """All-equal, quantised k/64 and underflowed-zero scores (tie-break = lowest flat index)."""
    O = oracle_mod
    z = load_golden("select_ties.npz")
    for name in ("equal", "quantised", "underflow", "random"):
        s64 = z[f"{name}_scores"]
        G, n = s64.shape
        s = T(s64, dtype, dev).reshape(1, -1)
        s64 = s.double().cpu().numpy().reshape(G, n)
        off = np.arange(G + 1) * n
        for k in (0, 1, 17, 400, 1203, G * n):
            r = A.segmented_select(s, off, k, "adaptive", want_raw=True)
            raw = O.adaptive_allocation(list(s64), k)
            if dtype == torch.float64:
                assert np.array_equal(raw, z[f"{name}_{k}_raw"])
            assert r["budgets"][0].cpu().tolist() == raw.tolist(), (name, k)
            keep = np.stack([O.topk_decision(s64[i], int(raw[i])) for i in range(G)])
            assert np.array_equal(r["keep"][0].cpu().numpy().reshape(G, n), keep), (name, k)
            for alpha in (0.0, 0.2, 1.0):
                rb = A.segmented_select(s, off, k, "adaptive", blend=True, alpha=alpha)
                assert rb["budgets"][0].cpu().tolist() == O.safeguard_blend(raw, k, G, alpha, np.full(G, n)).tolist()
        ks = z[f"{name}_topk_k"]
        rg = A.segmented_select(s, off, 0, "given", budgets=T(ks[None, :], torch.int32, dev))
        exp = np.stack([O.topk_decision(s64[i], int(ks[i])) for i in range(G)])
        assert np.array_equal(rg["keep"][0].cpu().numpy().reshape(G, n), exp), name


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_select_ragged_evict_rows(dev, oracle_mod, dtype):
    """evict_rows (policies.hpp:298-323) over ragged heads, several problems per launch."""
    O = oracle_mod
    rng = np.random.default_rng(11)
    for trial in range(12):
        S = int(rng.integers(1, 12))
        lens = rng.integers(1, 3000, size=S)
        off = np.concatenate([[0], np.cumsum(lens)])
        P = int(rng.integers(1, 4))
        rows64 = rng.exponential(size=(P, int(off[-1])))
        if trial % 3 == 0:
            rows64 = np.round(rows64 * 8) / 8  # heavy ties
        s = T(rows64, dtype, dev)
        s64 = s.double().cpu().numpy()
        total = int(rng.integers(S, int(off[-1]) + 1))
        alpha = float(rng.random())
        for adaptive in (True, False):
            r = A.segmented_select(s, off, total, "adaptive" if adaptive else "uniform", blend=adaptive,
                                   alpha=alpha, repair=True)
            for p in range(P):
                rows = [s64[p, off[i]:off[i + 1]] for i in range(S)]
                alloc, keep = O.evict_rows(rows, total, adaptive, alpha)
                assert r["budgets"][p].cpu().tolist() == alloc.tolist()
                assert np.array_equal(r["keep"][p].cpu().numpy(), np.concatenate(keep))
                kp = np.concatenate([np.nonzero(x)[0] for x in keep])
                assert np.array_equal(r["kept_pos"][p, :total].cpu().numpy(), kp)


def test_select_streaming(dev, oracle_mod):
    O = oracle_mod
    s = torch.rand(2, 8 * 100, device=dev, dtype=torch.float32)
    off = np.arange(9) * 100
    r = A.segmented_select(s, off, 200, "uniform", repair=True, streaming=True, sink_tokens=4)
    b = O.uniform_allocation(200, 8, np.full(8, 100))
    exp = np.concatenate([O.streaming_llm_decision(100, min(4, int(x)), int(x) - min(4, int(x))) for x in b])
    for p in range(2):
        assert np.array_equal(r["keep"][p].cpu().numpy(), exp)


# --------------------------------------------------------------------------- scoring
def _split_case(z, i):
    p = f"c{i}_"
    return (z[p + "q"], z[p + "k_out"], z[p + "v_out"], z[p + "k_win"], z[p + "v_win"], z[p + "params"].tolist(),
            float(z[p + "alpha"]))


def _kv(ko, kw):
    return np.concatenate([ko, kw], axis=1)[None]


def test_window_scores_fp64_vs_oracle(dev, oracle_mod):
    O = oracle_mod
    z = load_golden("evict_small.npz")
    for i in range(0, int(z["count"]), 5):
        q, ko, vo, kw, vw, (LB, pk, kind), alpha = _split_case(z, i)
        H, m, d = q.shape
        G, n, _ = ko.shape
        gs, hs = A.window_scores(T(q[None], torch.float64, dev), T(_kv(ko, kw), torch.float64, dev), pk,
                                 head_scores=True)
        ref = z[f"c{i}_group_scores"].reshape(G, n)
        tol = 1e-12 * np.abs(ref).max(axis=1, keepdims=True)
        assert np.all(np.abs(gs[0].cpu().numpy() - ref) <= tol), i
        for h in range(H):
            rh = O.window_scores(q[h], ko[h // (H // G)], pk)
            assert np.allclose(hs[0, h].cpu().numpy(), rh, rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("dtype,rel", [(torch.float32, 1e-5), (torch.bfloat16, 1e-4)])
def test_window_scores_llama_shape(dev, oracle_mod, dtype, rel):
    """Config-1 shape (32 Q / 8 KV heads, d=128, m=32, k=7, 4K prompt), planted heads."""
    O = oracle_mod
    q, k, v = planted_layer(1, 32, 8, 4064, 32, 128, seed=7, dtype=dtype, device=dev)
    gs = A.window_scores(q, k, 7)
    q64 = q.double().cpu().numpy()[0]
    k64 = k.double().cpu().numpy()[0]
    for g in (0, 3, 7):  # oracle cost: ~1 s per group
        per = [O.window_scores(q64[h], k64[g, :4064], 7) for h in range(g * 4, g * 4 + 4)]
        ref = O.group_mean_scores(np.stack(per), 4)[0]
        err = np.abs(gs[0, g].double().cpu().numpy() - ref).max()
        assert err <= rel * ref.max(), (g, err, ref.max())


# --------------------------------------------------------------------------- compress (evict_layer)
def test_compress_fp64_golden(dev, oracle_mod):
    """All 60 reference-generated evict_layer cases (5 kinds) through the full device pipeline."""
    O = oracle_mod
    z = load_golden("evict_small.npz")
    kinds = {v: k for k, v in O.KINDS.items()}
    for i in range(int(z["count"])):
        q, ko, vo, kw, vw, (LB, pk, kind), alpha = _split_case(z, i)
        H, m, d = q.shape
        G, n, _ = ko.shape
        out = A.compress(T(q[None], torch.float64, dev), T(_kv(ko, kw), torch.float64, dev),
                         T(_kv(vo, vw), torch.float64, dev), LB, kind=kinds[kind], pool_kernel=pk, alpha=alpha,
                         return_scores=True, return_keep=True)
        ref_scores = z[f"c{i}_group_scores"].reshape(G, n)
        assert np.all(np.abs(out.scores[0].cpu().numpy() - ref_scores) <= 1e-12 * np.abs(ref_scores).max()), i
        # identical-score gate: the oracle's selection on the GPU's scores == GPU selection
        r = O.evict_layer(q, ko, vo, kw, vw, LB, kind=kinds[kind], pool_kernel=pk, alpha=alpha)
        assert out.budgets.cpu().tolist() == z[f"c{i}_alloc"].tolist() == r.alloc.tolist(), i
        assert np.array_equal(out.keep[0].cpu().numpy().ravel(), z[f"c{i}_keep"]), i
        assert out.seqlens.cpu().tolist() == z[f"c{i}_ret_len"].tolist()
        rows = torch.cat([out.segment(0, g)[0] for g in range(G)]).cpu().numpy()
        vals = torch.cat([out.segment(0, g)[1] for g in range(G)]).cpu().numpy()
        assert np.array_equal(rows, z[f"c{i}_k_ret"]) and np.array_equal(vals, z[f"c{i}_v_ret"]), i


@pytest.mark.parametrize("kind", ["ada_snapkv", "snapkv", "streaming_llm"])
def test_compress_bf16_llama_identical_scores(dev, oracle_mod, kind):
    """bf16 Llama-shaped layers (P=2): GPU scores within tolerance of the oracle; the oracle's
    selection fed the GPU's own scores reproduces budgets, decisions and the packed rows bit-exactly."""
    O = oracle_mod
    P, H, G, m, n_o, d = 2, 32, 8, 32, 4064, 128
    LB = 1024 * G
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=3, dtype=torch.bfloat16, device=dev)
    out = A.compress(q, k, v, LB, kind=kind, pool_kernel=7, alpha=0.2, reserve=16, return_scores=True,
                     return_keep=True)
    torch.cuda.synchronize()
    outside = LB - m * G
    for p in range(P):
        s64 = out.scores[p].double().cpu().numpy()
        if kind == "ada_snapkv":
            raw, b, keep = _oracle_select(O, s64, outside, 0.2)
        else:
            b = O.repair_zero_budgets(O.uniform_allocation(outside, G, np.full(G, n_o)), np.full(G, n_o))
            if kind == "snapkv":
                keep = np.stack([O.topk_decision(s64[i], int(b[i])) for i in range(G)])
            else:
                keep = np.stack([O.streaming_llm_decision(n_o, min(4, int(x)), int(x) - min(4, int(x))) for x in b])
        assert out.budgets[p * G:(p + 1) * G].cpu().tolist() == b.tolist()
        assert np.array_equal(out.keep[p].cpu().numpy(), keep)
        kk = k[p].cpu()
        vv = v[p].cpu()
        for g in range(G):
            idx = np.concatenate([np.nonzero(keep[g])[0], n_o + np.arange(m)])
            kr, vr = out.segment(p, g)
            assert torch.equal(kr.cpu(), kk[g, idx]) and torch.equal(vr.cpu(), vv[g, idx])
    # scores vs the oracle on the same bf16 values (one group per problem; ~1 s each)
    q64, k64 = q.double().cpu().numpy(), k.double().cpu().numpy()
    for p in range(P):
        g = 5
        per = [O.window_scores(q64[p, h], k64[p, g, :n_o], 7) for h in range(g * 4, g * 4 + 4)]
        ref = O.group_mean_scores(np.stack(per), 4)[0]
        assert np.abs(out.scores[p, g].double().cpu().numpy() - ref).max() <= 1e-4 * ref.max()


def test_compress_host_resident_v_identical(dev):
    """V given as a pinned host tensor (the gather reads its retained and window rows over the
    host link): every output -- budgets, decisions and both cache planes -- is byte-identical
    to the device-V call; unpinned host memory is refused by the C ABI."""
    P, H, G, m, n_o, d = 2, 32, 8, 32, 4064, 128
    LB = 1024 * G
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=5, dtype=torch.bfloat16, device=dev)
    ref = A.compress(q, k, v, LB, reserve=8, return_keep=True)
    vh = v.cpu().pin_memory()
    got = A.compress(q, k, vh, LB, reserve=8, return_keep=True)
    torch.cuda.synchronize()
    for name in ("budgets", "seg_start", "seqlens", "keep"):
        assert torch.equal(getattr(got, name), getattr(ref, name)), name
    for p in range(P):  # the segments' rows (the reserve rows past them are unwritten)
        for g in range(G):
            (kr, vr), (kg, vg) = ref.segment(p, g), got.segment(p, g)
            assert torch.equal(kg, kr) and torch.equal(vg, vr)
    with pytest.raises(A.InvalidArgument):
        A.compress(q, k, v.cpu(), LB)
    import ctypes as C
    from paper_2407_11550_b200 import _lib
    plain = torch.zeros(16)
    dp = C.c_void_p()
    assert _lib.lib().adakv_host_device_pointer(C.c_void_p(plain.data_ptr()), C.byref(dp)) == 1  # invalid_argument


def test_compress_in_layer_chunks_identical(dev):
    """A model compressed in chunks of layers (pipeline.compress_model first_layer, as the
    e2e bench does while later layers are still arriving) fills the same cache as one call."""
    from paper_2407_11550_b200 import pipeline as PL
    Lyr, H, G, m, n_o, d = 4, 32, 8, 32, 1000, 128
    LB = 256 * G
    q, k, v = planted_layer(Lyr, H, G, n_o, m, d, seed=9, dtype=torch.bfloat16, device=dev)
    q, k, v = q.reshape(Lyr, 1, H, m, d), k.reshape(Lyr, 1, G, n_o + m, d), v.reshape(Lyr, 1, G, n_o + m, d)
    one = PL.compress_model(q, k, v, LB, reserve=4)
    ch = PL.compress_model(q, k, v, LB, reserve=4)
    ch.k.zero_()
    ch.seg_start.zero_()
    for l0 in (2, 0, 3, 1):  # any order
        PL.compress_model(q[l0:l0 + 1], k[l0:l0 + 1], v.cpu().pin_memory()[l0:l0 + 1], LB, reserve=4, out=ch,
                          first_layer=l0)
    torch.cuda.synchronize()
    for name in ("budgets", "seg_start", "seqlens"):
        assert torch.equal(getattr(ch, name), getattr(one, name)), name
    for p in range(Lyr):
        for g in range(G):
            (k1, v1), (k2, v2) = one.segment(p, g), ch.segment(p, g)
            assert torch.equal(k1, k2) and torch.equal(v1, v2)
    with pytest.raises(A.InvalidArgument):
        PL.compress_model(q[3:], k[3:], v[3:], LB, reserve=4, out=ch, first_layer=4)


def test_compress_per_problem_budgets(dev, oracle_mod):
    """pyramid schedule (budget.hpp:169-191): per-problem layer budgets in one launch."""
    O = oracle_mod
    P, H, G, m, n_o, d = 4, 8, 2, 4, 300, 16
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=5, dtype=torch.float32, device=dev)
    lbs = A.pyramid_layer_budgets(200, P, 1.5, 0.5) + m * G
    out = A.compress(q, k, v, 0, kind="ada_pyramid", layer_budgets=torch.tensor(lbs, device=dev),
                     return_scores=True, return_keep=True, reserve=3)
    for p in range(P):
        s64 = out.scores[p].double().cpu().numpy()
        raw, b, keep = _oracle_select(O, s64, int(lbs[p]) - m * G, 0.2)
        assert out.budgets[p * G:(p + 1) * G].cpu().tolist() == b.tolist()
        assert np.array_equal(out.keep[p].cpu().numpy(), keep)
    starts = out.seg_start.cpu().numpy()
    assert starts[0] == 0 and np.all(np.diff(starts) > 0)


# --------------------------------------------------------------------------- decode
def _cache_from_oracle(O, dev, dtype, rng, G=2, H=8, d=16, m=3, n=50, LB=40, reserve=4):
    q = rng.normal(size=(H, m, d))
    ko, vo = rng.normal(size=(G, n, d)), rng.normal(size=(G, n, d))
    kw, vw = rng.normal(size=(G, m, d)), rng.normal(size=(G, m, d))
    out = A.compress(T(q[None], dtype, dev), T(_kv(ko, kw), dtype, dev), T(_kv(vo, vw), dtype, dev), LB,
                     kind="ada_snapkv", pool_kernel=3, reserve=reserve)
    return out


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_decode_multistep_append_vs_oracle(dev, oracle_mod, dtype):
    O = oracle_mod
    rng = np.random.default_rng(4)
    G, H, d = 2, 8, 16
    cache = _cache_from_oracle(O, dev, dtype, rng, G=G, H=H, d=d)
    ws = torch.zeros(A.ops.decode_workspace_bytes(1, H, G, d, cache.max_rows + 8), dtype=torch.uint8, device=dev)
    segs = [[x.double().cpu().numpy() for x in cache.segment(0, g)] for g in range(G)]
    for step in range(4):
        qd = rng.normal(size=(H, d))
        kn, vn = rng.normal(size=(G, d)), rng.normal(size=(G, d))
        kn = torch.as_tensor(kn).to(dtype).double().numpy()  # the cache stores `dtype`
        vn = torch.as_tensor(vn).to(dtype).double().numpy()
        qd = torch.as_tensor(qd).to(dtype).double().numpy()
        o = A.decode(T(qd[None], dtype, dev), cache, T(kn[None], dtype, dev), T(vn[None], dtype, dev),
                     max_rows=cache.max_rows + 8, ws=ws)
        for g in range(G):  # append_kv: the new row goes last (attention.hpp:126-134)
            segs[g][0] = np.vstack([segs[g][0], kn[g]])
            segs[g][1] = np.vstack([segs[g][1], vn[g]])
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd, np.vstack([s[0] for s in segs]), np.vstack([s[1] for s in segs]), off)
        tol = 1e-12 if dtype == torch.float64 else 2e-5
        assert np.abs(o[0].double().cpu().numpy() - ref).max() <= tol * max(1.0, np.abs(ref).max())
        assert cache.seqlens.cpu().tolist() == [s[0].shape[0] for s in segs]
        for g in range(G):
            kr, vr = cache.segment(0, g)
            assert np.array_equal(kr.double().cpu().numpy(), segs[g][0])


def test_decode_bf16_llama_shape(dev, oracle_mod):
    O = oracle_mod
    P, H, G, m, n_o, d = 2, 32, 8, 32, 4064, 128
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=9, dtype=torch.bfloat16, device=dev)
    cache = A.compress(q, k, v, 1024 * G, reserve=8)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    qd = torch.randn((P, H, d), generator=gen, device=dev).to(torch.bfloat16)
    o = A.decode(qd, cache)
    for p in range(P):
        segs = [cache.segment(p, g) for g in range(G)]
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd[p].double().cpu().numpy(), torch.cat([s[0] for s in segs]).double().cpu().numpy(),
                                 torch.cat([s[1] for s in segs]).double().cpu().numpy(), off)
        err = np.abs(o[p].double().cpu().numpy() - ref).max()
        assert err <= 2e-2 and err <= 1e-2 * max(np.abs(ref).max(), 1e-3) + 4e-3, err


def test_device_error_latch(dev):
    """topk_decision k > n (policies.hpp:83) detected on the device -> InvalidArgument."""
    s = torch.rand(1, 10, device=dev)
    r = A.segmented_select(s, [0, 5, 10], 0, "given", budgets=torch.tensor([[6, 1]], dtype=torch.int32, device=dev))
    with pytest.raises(A.InvalidArgument):
        A.workspace_status(r["ws"])


# --------------------------------------------------------------------------- question-agnostic glue
def test_question_agnostic_append_then_decode(dev, oracle_mod):
    """Config-5 flow: compress on the context window, append T question rows per segment with
    adakv_append_rows (bit-exact copies after the window rows), then decode over the result."""
    from paper_2407_11550_b200 import pipeline as PL
    O = oracle_mod
    Lyr, B, H, G, m, n_o, d, T = 2, 2, 32, 8, 32, 2016, 128, 16
    q, k, v = planted_layer(Lyr * B, H, G, n_o, m, d, seed=23, dtype=torch.bfloat16, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    kq = torch.randn((Lyr, B, G, T, d), generator=gen, device=dev).to(torch.bfloat16)
    vq = torch.randn((Lyr, B, G, T, d), generator=gen, device=dev).to(torch.bfloat16)
    LB = 256 * G
    cache = PL.compress_question_agnostic(q.view(Lyr, B, H, m, d), k.view(Lyr, B, G, n_o + m, d),
                                          v.view(Lyr, B, G, n_o + m, d), LB, kq, vq, reserve=T + 4)
    plain = A.compress(q, k, v, LB, reserve=T + 4)
    budgets = plain.budgets.cpu().numpy()
    for p in range(Lyr * B):
        for g in range(G):
            kr, vr = cache.segment(p, g)
            k0, v0 = plain.segment(p, g)
            assert kr.shape[0] == int(budgets[p * G + g]) + m + T
            assert torch.equal(kr[:-T], k0) and torch.equal(vr[:-T], v0)
            assert torch.equal(kr[-T:], kq.view(-1, G, T, d)[p, g]) and torch.equal(vr[-T:], vq.view(-1, G, T, d)[p, g])
    qd = torch.randn((Lyr * B, H, d), generator=gen, device=dev).to(torch.bfloat16)
    o = A.decode(qd, cache)
    for p in (0, 3):
        segs = [cache.segment(p, g) for g in range(G)]
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd[p].double().cpu().numpy(), torch.cat([s[0] for s in segs]).double().cpu().numpy(),
                                 torch.cat([s[1] for s in segs]).double().cpu().numpy(), off)
        err = np.abs(o[p].double().cpu().numpy() - ref).max()
        assert err <= 2e-2, err


def test_pyramid_problem_budgets_layer_major(dev, oracle_mod):
    from paper_2407_11550_b200 import pipeline as PL
    O = oracle_mod
    lb = PL.pyramid_problem_budgets(1000, 4, 3, G=8, m=32)
    sched = O.pyramid_layer_budgets(1000, 4, 1.5, 0.5)
    assert lb.tolist() == [int(x) + 256 for x in np.repeat(sched, 3)]


def test_decode_graph_pdl_chain_matches_serial(dev):
    """The bench path: one CUDA graph per decode step over all layers, consecutive layers
    overlapped by programmatic dependent launch (each layer's cache streams in before the
    previous layer's decode has finished).  Every step's outputs and the appended caches must
    equal the serial, non-overlapped launches bit for bit."""
    from paper_2407_11550_b200 import pipeline as PL
    Lyr, B, H, G, m, n_o, d = 4, 1, 32, 8, 32, 4064, 128
    q, k, v = planted_layer(Lyr * B, H, G, n_o, m, d, seed=29, dtype=torch.bfloat16, device=dev)
    LB = 1024 * G
    steps = 5
    gen = torch.Generator(device=dev)
    gen.manual_seed(8)
    qs = torch.randn((steps, Lyr, B, H, d), generator=gen, device=dev).to(torch.bfloat16)
    ks = torch.randn((steps, Lyr, B, G, d), generator=gen, device=dev).to(torch.bfloat16)
    vs = torch.randn((steps, Lyr, B, G, d), generator=gen, device=dev).to(torch.bfloat16)
    outs = {}
    L = A.lib()
    for mode in ("graph_pdl", "serial"):
        cache = PL.compress_model(q.view(Lyr, B, H, m, d), k.view(Lyr, B, G, n_o + m, d), v.view(Lyr, B, G, n_o + m, d),
                                  LB, reserve=steps + 1)
        prev = L.adakv_set_decode_overlap(1 if mode == "graph_pdl" else 0)
        try:
            dg = PL.DecodeGraph(cache, Lyr, B, LB + steps + 1, use_graph=(mode == "graph_pdl"))
            res = []
            for s in range(steps):
                dg.q.copy_(qs[s])
                dg.k_new.copy_(ks[s])
                dg.v_new.copy_(vs[s])
                res.append(dg.step().clone())
            torch.cuda.synchronize()
        finally:
            L.adakv_set_decode_overlap(prev)
        segs = [torch.cat(cache.segment(p, g)) for p in range(Lyr * B) for g in range(G)]  # valid rows only
        outs[mode] = (torch.stack(res), segs, cache.seqlens.clone())
    a, b = outs["graph_pdl"], outs["serial"]
    assert torch.equal(a[2], b[2])
    assert int(a[2][0]) == int(b[2][0]) and torch.equal(a[0], b[0])
    assert all(torch.equal(x, y) for x, y in zip(a[1], b[1]))


def test_decode_long_segments_ring_rounds(dev, oracle_mod):
    """Segments far longer than a CTA's TMA ring (every slot refilled several times) and a
    few decode steps with appends, against the fp64 oracle."""
    O = oracle_mod
    P, H, G, m, n_o, d = 1, 32, 8, 32, 32736, 128
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=31, dtype=torch.bfloat16, device=dev)
    LB = 16384 * G  # half of every group's keys retained: ~16K rows per segment
    cache = A.compress(q, k, v, LB, reserve=4)
    gen = torch.Generator(device=dev)
    gen.manual_seed(12)
    for step in range(3):
        qd = torch.randn((P, H, d), generator=gen, device=dev).to(torch.bfloat16)
        kn = torch.randn((P, G, d), generator=gen, device=dev).to(torch.bfloat16)
        vn = torch.randn((P, G, d), generator=gen, device=dev).to(torch.bfloat16)
        o = A.decode(qd, cache, kn, vn)
        segs = [cache.segment(0, g) for g in range(G)]  # include the appended row
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd[0].double().cpu().numpy(), torch.cat([s[0] for s in segs]).double().cpu().numpy(),
                                 torch.cat([s[1] for s in segs]).double().cpu().numpy(), off)
        err = np.abs(o[0].double().cpu().numpy() - ref).max()
        assert err <= 2e-2 and err <= 1e-2 * max(np.abs(ref).max(), 1e-3) + 4e-3, (step, err)
        assert torch.equal(segs[3][0][-1], kn[0, 3]) and torch.equal(segs[3][1][-1], vn[0, 3])


def test_decode_three_block_warps_vs_oracle(dev, oracle_mod):
    """Segment lengths that give warps exactly three 16-row blocks (the fused three-block step)
    or a pair followed by a single, with appends, against the fp64 oracle."""
    from paper_2407_11550_b200.ops import CompressedCache
    O = oracle_mod
    P, H, G, d, reserve = 1, 32, 8, 128, 4
    lens = np.array([3455, 2879, 2300, 1000, 47, 3456 + 16 * 9 - 1, 3000, 2049], dtype=np.int32)
    caps = lens + reserve
    starts = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int32)
    rows = int(caps.sum())
    gen = torch.Generator(device=dev)
    gen.manual_seed(21)
    kp = (torch.randn((rows, d), generator=gen, device=dev) * 0.5).to(torch.bfloat16)
    vp = torch.randn((rows, d), generator=gen, device=dev).to(torch.bfloat16)
    cache = CompressedCache(k=kp, v=vp, seg_start=torch.as_tensor(starts, device=dev),
                            seqlens=torch.as_tensor(lens, device=dev), budgets=torch.as_tensor(lens, device=dev),
                            P=P, H=H, G=G, m=0, d=d, reserve=reserve, layer_budget=int(lens.max()))
    for step in range(2):
        qd = torch.randn((P, H, d), generator=gen, device=dev).to(torch.bfloat16)
        kn = torch.randn((P, G, d), generator=gen, device=dev).to(torch.bfloat16)
        vn = torch.randn((P, G, d), generator=gen, device=dev).to(torch.bfloat16)
        o = A.decode(qd, cache, kn, vn)
        segs = [cache.segment(0, g) for g in range(G)]
        assert [sg[0].shape[0] for sg in segs] == (lens + step + 1).tolist()
        off = np.concatenate([[0], np.cumsum([sg[0].shape[0] for sg in segs])])
        ref = O.decode_attention(qd[0].double().cpu().numpy(), torch.cat([sg[0] for sg in segs]).double().cpu().numpy(),
                                 torch.cat([sg[1] for sg in segs]).double().cpu().numpy(), off)
        err = np.abs(o[0].double().cpu().numpy() - ref).max()
        assert err <= 2e-2 and err <= 1e-2 * max(np.abs(ref).max(), 1e-3) + 4e-3, (step, err)
        for g in range(G):
            assert torch.equal(segs[g][0][-1], kn[0, g]) and torch.equal(segs[g][1][-1], vn[0, g])


@pytest.mark.parametrize("H,G", [(2, 2), (4, 2), (6, 2), (8, 2), (10, 2), (12, 2), (14, 2), (16, 2)])
def test_decode_bf16_group_sizes_append(dev, oracle_mod, H, G):
    """The tensor-core decode at every group size g = H/G in 1..8 (head quads, padded heads,
    the CTA merge's (warp, head) lanes), two steps with appends: outputs within the bf16
    tolerance of the fp64 oracle, the appended rows and lengths exact."""
    from paper_2407_11550_b200.ops import CompressedCache
    O = oracle_mod
    rng = np.random.default_rng(H * 10 + G)
    d, steps = 128, 2
    lens = rng.integers(150, 700, size=G).astype(np.int32)
    caps = lens + steps + 2
    starts = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int32)
    rows = int(caps.sum())
    kp = torch.as_tensor(rng.normal(size=(rows, d)) * 0.5).to(torch.bfloat16).to(dev)
    vp = torch.as_tensor(rng.normal(size=(rows, d))).to(torch.bfloat16).to(dev)
    cache = CompressedCache(k=kp, v=vp, seg_start=torch.as_tensor(starts, device=dev),
                            seqlens=torch.as_tensor(lens, device=dev), budgets=torch.as_tensor(lens, device=dev),
                            P=1, H=H, G=G, m=0, d=d, reserve=steps + 2, layer_budget=int(lens.sum()))
    segs = [[x.double().cpu().numpy() for x in cache.segment(0, g)] for g in range(G)]
    for step in range(steps):
        qd = torch.as_tensor(rng.normal(size=(1, H, d))).to(torch.bfloat16).to(dev)
        kn = torch.as_tensor(rng.normal(size=(1, G, d))).to(torch.bfloat16).to(dev)
        vn = torch.as_tensor(rng.normal(size=(1, G, d))).to(torch.bfloat16).to(dev)
        o = A.decode(qd, cache, kn, vn, max_rows=int(caps.max()))
        for g in range(G):
            segs[g][0] = np.vstack([segs[g][0], kn[0, g].double().cpu().numpy()])
            segs[g][1] = np.vstack([segs[g][1], vn[0, g].double().cpu().numpy()])
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd[0].double().cpu().numpy(), np.vstack([s[0] for s in segs]),
                                 np.vstack([s[1] for s in segs]), off)
        err = np.abs(o[0].double().cpu().numpy() - ref).max()
        assert err <= 2e-2 and err <= 1e-2 * max(np.abs(ref).max(), 1e-3) + 4e-3, (step, err)
        assert cache.seqlens.cpu().tolist() == [s[0].shape[0] for s in segs]
        for g in range(G):
            kr, vr = cache.segment(0, g)
            assert np.array_equal(kr.double().cpu().numpy(), segs[g][0])
            assert np.array_equal(vr.double().cpu().numpy(), segs[g][1])


def test_decode_bf16_tiny_and_empty_segments_append(dev, oracle_mod):
    """Segments of 0..40 rows (empty before the append, single partial blocks, most warps and
    CTAs without blocks): three appended steps, outputs within tolerance, rows exact."""
    from paper_2407_11550_b200.ops import CompressedCache
    O = oracle_mod
    rng = np.random.default_rng(11)
    H, G, d, steps = 32, 8, 128, 3
    lens = np.array([0, 1, 2, 15, 16, 17, 31, 40], dtype=np.int32)
    caps = lens + steps + 1
    starts = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int32)
    rows = int(caps.sum())
    kp = torch.as_tensor(rng.normal(size=(rows, d)) * 0.5).to(torch.bfloat16).to(dev)
    vp = torch.as_tensor(rng.normal(size=(rows, d))).to(torch.bfloat16).to(dev)
    cache = CompressedCache(k=kp, v=vp, seg_start=torch.as_tensor(starts, device=dev),
                            seqlens=torch.as_tensor(lens, device=dev), budgets=torch.as_tensor(lens, device=dev),
                            P=1, H=H, G=G, m=0, d=d, reserve=steps + 1, layer_budget=int(lens.sum()))
    segs = [[x.double().cpu().numpy() for x in cache.segment(0, g)] for g in range(G)]
    for step in range(steps):
        qd = torch.as_tensor(rng.normal(size=(1, H, d))).to(torch.bfloat16).to(dev)
        kn = torch.as_tensor(rng.normal(size=(1, G, d))).to(torch.bfloat16).to(dev)
        vn = torch.as_tensor(rng.normal(size=(1, G, d))).to(torch.bfloat16).to(dev)
        o = A.decode(qd, cache, kn, vn, max_rows=int(caps.max()))
        for g in range(G):
            segs[g][0] = np.vstack([segs[g][0], kn[0, g].double().cpu().numpy()])
            segs[g][1] = np.vstack([segs[g][1], vn[0, g].double().cpu().numpy()])
        off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
        ref = O.decode_attention(qd[0].double().cpu().numpy(), np.vstack([s[0] for s in segs]),
                                 np.vstack([s[1] for s in segs]), off)
        err = np.abs(o[0].double().cpu().numpy() - ref).max()
        assert err <= 2e-2 and err <= 1e-2 * max(np.abs(ref).max(), 1e-3) + 4e-3, (step, err)
        assert cache.seqlens.cpu().tolist() == [s[0].shape[0] for s in segs]
        for g in range(G):
            kr, vr = cache.segment(0, g)
            assert np.array_equal(kr.double().cpu().numpy(), segs[g][0])
            assert np.array_equal(vr.double().cpu().numpy(), segs[g][1])
