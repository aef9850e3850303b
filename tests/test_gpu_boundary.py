"""GPU checks of the boundary's device-side contract: what the reference throws for
(LayerCache::validate attention.hpp:76-83, append_kv attention.hpp:126-134, the evict_layer
budget floor policies.hpp:229-231 and apportion's capacity budget.hpp:48-59) is latched on the
device and raised through workspace_status with the reference's message -- and nothing is
written out of bounds on the way.  Plus the selection kernel's rank ranges at cluster slice
boundaries that do not divide the element count.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200 import _lib as L  # noqa: E402
from paper_2407_11550_b200 import ops  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402


@pytest.mark.parametrize("off", [[0, 13334, 40000], [0, 13333, 40000], [0, 26666, 26667, 40000],
                                 [0, 1, 13333, 13334, 26667, 40000], [0, 0, 40000, 40000]])
def test_select_segments_ending_on_cluster_slice_boundaries(dev, oracle_mod, off):
    """N = 40000 keys take a 3-CTA cluster whose slices [0,13333), [13333,26666), [26666,40000)
    do not divide N: segments that start or end on an element next to a slice boundary must be
    counted by the rank that owns it (adaptive, blended and per-segment selections bit-exact)."""
    O = oracle_mod
    rng = np.random.default_rng(len(off))
    off = np.asarray(off, np.int64)
    S = off.size - 1
    s = torch.as_tensor(np.round(rng.exponential(size=(2, 40000)) * 16) / 16, dtype=torch.float32, device=dev)
    s64 = s.double().cpu().numpy()
    nonempty = int((np.diff(off) > 0).sum())
    for total in (nonempty, 777, 13334, 39999, 40000):
        r = A.segmented_select(s, off, total, "adaptive", want_raw=True)
        for p in range(2):
            rows = [s64[p, off[i]:off[i + 1]] for i in range(S)]
            raw = O.adaptive_allocation(rows, total)
            assert r["budgets"][p].cpu().tolist() == raw.tolist(), (total, p)
            keep = np.concatenate([O.topk_decision(rows[i], int(raw[i])) for i in range(S)])
            assert np.array_equal(r["keep"][p].cpu().numpy(), keep)
            kp = np.concatenate([np.nonzero(O.topk_decision(rows[i], int(raw[i])))[0] for i in range(S)])
            assert np.array_equal(r["kept_pos"][p, :total].cpu().numpy(), kp)
        A.workspace_status(r["ws"])


def bits(t):
    # reserved rows are uninitialised: compare (and copy) bit patterns -- a bf16 copy may
    # canonicalise NaN payloads, and NaN != NaN
    return t.view(torch.int16)


def _layer(dev, seed=3, P=1, H=8, G=2, n_o=1000, m=32, d=128):
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=seed, dtype=torch.bfloat16, device=dev)
    return q, k, v


def test_nonfinite_key_in_window_statistics_raises(dev):
    q, k, v = _layer(dev)
    k[0, 1, 17, 5] = float("nan")  # an outside key: every window row's softmax sum turns NaN
    with pytest.raises(A.InvalidArgument, match="non-finite"):
        A.compress(q, k, v, 128 * 2, check=True)


def test_nonfinite_value_in_retained_row_raises(dev):
    q, k, v = _layer(dev)
    v[0, 0, -1, 3] = float("inf")  # a window row: always retained, so the gather copies it
    with pytest.raises(A.InvalidArgument, match="non-finite"):
        A.compress(q, k, v, 128 * 2, check=True)


def test_nonfinite_in_evicted_row_needs_the_full_scan(dev):
    """An evicted V row is never read by the compress path; validate=True scans all of K and V
    (the reference's LayerCache::validate) and raises for it."""
    q, k, v = _layer(dev)
    c = A.compress(q, k, v, 64 * 2, return_keep=True, check=True)
    keep = c.keep[0, 0].cpu().numpy()
    pos = int(np.nonzero(keep == 0)[0][0])
    v[0, 0, pos, 0] = float("nan")
    A.compress(q, k, v, 64 * 2, check=True)  # evicted: not seen, identical result
    with pytest.raises(A.InvalidArgument, match="non-finite"):
        A.compress(q, k, v, 64 * 2, validate=True, check=True)


def test_decode_append_past_capacity_is_refused_and_raised(dev):
    q, k, v = _layer(dev)
    G, d = 2, 128
    cache = A.compress(q, k, v, 128 * G, reserve=1)
    assert cache.seg_cap.cpu().tolist() == (cache.seqlens + 1).cpu().tolist()
    planes = (bits(cache.k).clone(), bits(cache.v).clone())
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    qd = torch.randn((1, 8, d), generator=gen, device=dev).to(torch.bfloat16)
    kn = torch.randn((1, G, d), generator=gen, device=dev).to(torch.bfloat16)
    ws = torch.zeros(ops.decode_workspace_bytes(1, 8, G, d, cache.max_rows + 2), dtype=torch.uint8, device=dev)
    A.decode(qd, cache, kn, kn, ws=ws, check=True)  # fills the one reserved row
    L0 = cache.seqlens.clone()
    k1, v1 = bits(cache.k).clone(), bits(cache.v).clone()
    o_full = A.decode(qd, cache, None, None, ws=ws, check=True)
    o = A.decode(qd, cache, kn * 2, kn * 2, ws=ws)  # no room: refused, attends the existing rows
    with pytest.raises(A.InvalidArgument, match="capacity exhausted"):
        A.workspace_status(ws)
    assert torch.equal(cache.seqlens, L0)
    assert torch.equal(bits(cache.k), k1) and torch.equal(bits(cache.v), v1)  # nothing written anywhere
    assert torch.equal(o, o_full)
    # the rows of the first step landed in each segment's reserved row, nowhere else
    changed = (k1 != planes[0]).any(dim=1).nonzero().flatten().cpu().tolist()
    assert changed == [int(s) + int(n) - 1 for s, n in zip(cache.seg_start.cpu(), cache.seqlens.cpu())]


def test_append_rows_past_capacity_is_refused_and_raised(dev):
    q, k, v = _layer(dev)
    G, d = 2, 128
    cache = A.compress(q, k, v, 128 * G, reserve=3)
    rows = torch.ones((G, 4, d), dtype=torch.bfloat16, device=dev)
    k0 = bits(cache.k).clone()
    with pytest.raises(A.InvalidArgument, match="capacity exhausted"):
        A.append_rows(cache, rows, rows)
    assert torch.equal(bits(cache.k), k0)
    A.append_rows(cache, rows[:, :3], rows[:, :3])  # exactly fills the reserve
    with pytest.raises(A.InvalidArgument, match="capacity exhausted"):
        A.append_kv(cache, rows[:, 0], rows[:, 0])


def test_per_problem_budgets_outside_floor_or_capacity(dev):
    """The pyramid path's per-problem layer budgets: ops.compress raises before launching, and a
    direct C-ABI caller gets the error latched with all budgets zero (no garbage layout)."""
    P, H, G, m, n_o, d = 3, 8, 2, 32, 1000, 128
    q, k, v = _layer(dev, P=P)
    for bad in ([100, 200, m * G + G - 1], [100, 200, G * n_o + m * G + 1]):
        lb = torch.tensor(bad, dtype=torch.int64, device=dev)
        with pytest.raises(A.InvalidArgument):
            A.compress(q, k, v, 0, layer_budgets=lb)
        shape = ops.layer_shape(P, H, G, m, n_o, d)
        cfg = ops.policy_config("ada_pyramid", 7, 0.2, 4, H // G, True, m)
        lib = L.lib()
        nb = C.c_size_t()
        L.check(lib.adakv_compress_workspace(L.BF16, C.byref(shape), C.byref(cfg), C.byref(nb)))
        ws = torch.zeros(nb.value, dtype=torch.uint8, device=dev)
        rows = P * G * (n_o + m)
        kc = torch.zeros((rows, d), dtype=torch.bfloat16, device=dev)
        vc = torch.zeros_like(kc)
        ss, sl, cap, bud = (torch.full((P * G,), -7, dtype=torch.int32, device=dev) for _ in range(4))
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        L.check(lib.adakv_compress(L.BF16, C.byref(shape), C.byref(cfg), 0, p(lb), p(q), p(k), p(v), 0, p(kc), p(vc),
                                   p(ss), p(sl), p(cap), p(bud), None, None, p(ws), ws.numel(),
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        with pytest.raises(A.InvalidArgument):
            A.workspace_status(ws)
        b = bud.view(P, G).cpu()
        assert (b[2] == 0).all()  # the rejected problem: zero budgets, window rows only
        assert (sl.view(P, G).cpu()[2] == m).all()


def test_decode_workspace_reuse_across_layouts(dev, oracle_mod):
    """ops.decode's cached workspace: a split-K decode of a small batch, then one of a larger
    batch (whose ticket words would land on the first call's partials) -- both exact."""
    O = oracle_mod
    for P in (3, 40, 3):
        q, k, v = planted_layer(P, 8, 8, 300, 8, 16, seed=P, dtype=torch.float64, device=dev)
        cache = A.compress(q, k, v, 64 * 8)
        qd = q[:, :, -1, :].contiguous()
        o = A.decode(qd, cache)
        for p in (0, P - 1):
            segs = [cache.segment(p, g) for g in range(8)]
            off = np.concatenate([[0], np.cumsum([s[0].shape[0] for s in segs])])
            ref = O.decode_attention(qd[p].cpu().numpy(), torch.cat([s[0] for s in segs]).cpu().numpy(),
                                     torch.cat([s[1] for s in segs]).cpu().numpy(), off)
            assert np.allclose(o[p].cpu().numpy(), ref, rtol=1e-10, atol=1e-12), (P, p)


@pytest.mark.parametrize("host_v", [False, True])
def test_compress_split_gather_chunks_match_one_call(dev, host_v):
    """adakv_compress_split: a model compressed in layer chunks with every chunk's gather forked
    onto a second stream (two alternating workspaces, joined before use) -- with V on the device
    or in pinned host memory -- writes exactly the cache one adakv_compress call writes."""
    from paper_2407_11550_b200 import pipeline as PL
    Lyr, B, H, G, m, n, d = 8, 1, 32, 8, 32, 1056, 128
    q, k, v = planted_layer(Lyr * B, H, G, n - m, m, d, seed=23, dtype=torch.bfloat16, device=dev)
    q, k, v = q.view(Lyr, B, H, m, d), k.view(Lyr, B, G, n, d), v.view(Lyr, B, G, n, d)
    LB = 128 * G
    ref = PL.compress_model(q, k, v, LB, reserve=3)
    out = PL.compress_model(q, k, v, LB, reserve=3)
    for t in (out.k, out.v):
        t.zero_()
    for t in (out.seg_start, out.seqlens, out.seg_cap, out.budgets):
        t.fill_(-7)
    vv = v.cpu().pin_memory() if host_v else v
    comp, gst = torch.cuda.current_stream(), torch.cuda.Stream(device=dev)
    nch, lc = 4, Lyr // 4
    wsb = ops.compress_workspace_bytes(q[:lc].reshape(lc * B, H, m, d), k[:lc].reshape(lc * B, G, n, d))
    wss = [torch.zeros(wsb, dtype=torch.uint8, device=dev) for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    for c in range(nch):
        if c >= 2:
            comp.wait_event(done[c & 1])
        sl = slice(c * lc, (c + 1) * lc)
        PL.compress_model(q[sl], k[sl], vv[sl], LB, reserve=3, out=out, first_layer=c * lc, ws=wss[c & 1],
                          gather_stream=gst)
        done[c & 1].record(gst)
    comp.wait_stream(gst)
    for name in ("seg_start", "seqlens", "seg_cap", "budgets"):
        assert torch.equal(getattr(out, name), getattr(ref, name)), name
    st, ln = ref.seg_start.cpu().numpy(), ref.seqlens.cpu().numpy()
    rows = torch.as_tensor(np.concatenate([np.arange(a, a + b) for a, b in zip(st, ln)]), device=dev)
    assert torch.equal(out.k[rows].view(torch.int16), ref.k[rows].view(torch.int16))
    assert torch.equal(out.v[rows].view(torch.int16), ref.v[rows].view(torch.int16))
    for w in wss:
        ops.workspace_status(w)
    with pytest.raises(L.InvalidArgument):
        ops.compress(q[0], k[0], v[0], LB, gather_stream=gst, check=True)


@pytest.mark.parametrize("cs", [None, "4"])
@pytest.mark.parametrize("seg", [[0, 300000], list(np.linspace(0, 300000, 9).astype(int)),
                                 [0, 7, 140001, 140002, 299990, 300000]])
def test_select_sixteen_cta_cluster_matches_oracle(dev, oracle_mod, seg, cs, monkeypatch):
    """A problem of 300K keys (one problem per call) takes a 16-CTA cluster (keys cached in
    shared memory): DSMEM histogram sums over more than eight ranks, ragged segments across rank
    boundaries.  Forced to 4 CTAs (ADAKV_SELECT_CS) the 75K-key slices are read from global
    memory instead.  Blended adaptive budgets and keep masks bit-exact to evict_rows."""
    if cs is not None:
        monkeypatch.setenv("ADAKV_SELECT_CS", cs)
    O = oracle_mod
    rng = np.random.default_rng(len(seg))
    off = np.asarray(seg, np.int64)
    S = off.size - 1
    x = np.round(rng.exponential(size=(1, 300000)) * 64) / 64  # heavy ties
    s = torch.as_tensor(x, dtype=torch.float32, device=dev)
    rows = [x[0, off[i]:off[i + 1]] for i in range(S)]
    for total in (S + 5, 20000, 150001):
        r = A.segmented_select(s, off, total, "adaptive", blend=True, alpha=0.2, repair=True)
        alloc, keep = O.evict_rows(rows, total, True, 0.2)
        assert r["budgets"][0].cpu().tolist() == alloc.tolist(), total
        assert np.array_equal(r["keep"][0].cpu().numpy(), np.concatenate(keep)), total
        kp = np.concatenate([np.nonzero(k)[0] for k in keep])
        assert np.array_equal(r["kept_pos"][0, :total].cpu().numpy(), kp), total
        A.workspace_status(r["ws"])


def test_select_many_segments_match_oracle(dev, oracle_mod):
    """40 and 64 segments per problem (MHA models: Llama-2-13B has 40 KV heads, 64-head models)
    take the lean shared-memory layout (one histogram buffer, no kept first-digit histogram):
    adaptive + blended budgets and keep masks bit-exact to evict_rows; 39 keep the full layout."""
    O = oracle_mod
    rng = np.random.default_rng(4)
    for S in (39, 40, 64):
        n = 1500
        x = np.round(rng.exponential(size=(2, S * n)) * 32) / 32
        s = torch.as_tensor(x, dtype=torch.float32, device=dev)
        off = np.arange(S + 1) * n
        for total in (S + 3, 20 * S, 700 * S):
            r = A.segmented_select(s, off, total, "adaptive", blend=True, alpha=0.2, repair=True)
            for p in range(2):
                rows = [x[p, off[i]:off[i + 1]] for i in range(S)]
                alloc, keep = O.evict_rows(rows, total, True, 0.2)
                assert r["budgets"][p].cpu().tolist() == alloc.tolist(), (S, total, p)
                assert np.array_equal(r["keep"][p].cpu().numpy(), np.concatenate(keep)), (S, total, p)
            A.workspace_status(r["ws"])


def test_compress_mha_40_kv_heads_on_own_scores(dev, oracle_mod):
    """A multi-head (no GQA) layer with 40 KV heads -- Llama-2-13B's attention -- through
    adakv_compress: the 40-segment selection (lean layout) on the device's own window scores
    equals evict_rows on those scores, and the cache holds exactly the kept rows."""
    O = oracle_mod
    P, H, G, m, n_o, d = 2, 40, 40, 32, 992, 128
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=13, dtype=torch.bfloat16, device=dev)
    LB = 160 * G + m * G
    c = A.compress(q, k, v, LB, return_scores=True, return_keep=True, check=True)
    sc = c.scores.double().cpu().numpy()
    for p in range(P):
        rows = [sc[p, g] for g in range(G)]
        alloc, keep = O.evict_rows(rows, LB - m * G, True, 0.2)
        assert c.budgets.view(P, G)[p].cpu().tolist() == alloc.tolist(), p
        assert np.array_equal(c.keep[p].cpu().numpy().ravel(), np.concatenate(keep)), p
        st, ln = c.seg_start.view(P, G)[p].cpu().numpy(), c.seqlens.view(P, G)[p].cpu().numpy()
        for g in range(0, G, 7):
            pos = np.nonzero(keep[g])[0]
            want = torch.cat([k[p, g, torch.as_tensor(pos, device=dev)], k[p, g, n_o:]])
            assert ln[g] == len(pos) + m
            assert torch.equal(bits(c.k[st[g]:st[g] + ln[g]]), bits(want)), (p, g)
