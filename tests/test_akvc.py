"""AKVC v1 export / import of compressed caches (flat_cache.hpp:131-178), SURVEY §8(f) item 2.

CPU: the reference's golden bytes (flat_cache_test.cpp:182-198) and malformed-input errors.
GPU: an fp64 compressed layer exported per query head equals the reference layout built from
the oracle's evict_layer result byte for byte; an imported file decodes like the original.
"""
import struct

import numpy as np
import pytest
import torch

from paper_2407_11550_b200 import akvc
from paper_2407_11550_b200._lib import FormatError, OutOfRange
from paper_2407_11550_b200.ops import CompressedCache


def _cpu_cache(rows_k, rows_v, G, H, seg_lens):
    d = rows_k.shape[1]
    starts = np.concatenate([[0], np.cumsum(seg_lens)[:-1]]).astype(np.int32)
    return CompressedCache(k=torch.as_tensor(rows_k), v=torch.as_tensor(rows_v),
                           seg_start=torch.as_tensor(starts), seqlens=torch.as_tensor(np.asarray(seg_lens, np.int32)),
                           budgets=torch.as_tensor(np.asarray(seg_lens, np.int32)), P=1, H=H, G=G, m=0, d=d,
                           reserve=0, layer_budget=int(sum(seg_lens)))


def test_golden_bytes_one_head():
    # flat_cache_test.cpp:182-198: one head, one row, d_h = 1, K = 1.5, V = -2.0 -> 40 bytes
    c = _cpu_cache(np.array([[1.5]]), np.array([[-2.0]]), G=1, H=1, seg_lens=[1])
    b = akvc.export_akvc(c)
    assert len(b) == 40 and b[:4] == b"AKVC"
    assert struct.unpack_from("<III", b, 4) == (1, 1, 1) and struct.unpack_from("<Q", b, 16) == (1,)
    assert b[24 + 7] == 0x3F and struct.unpack_from("<dd", b, 24) == (1.5, -2.0)


def test_per_query_head_layout_and_round_trip():
    rng = np.random.default_rng(0)
    lens = [3, 5]
    k = rng.normal(size=(8, 4))
    v = rng.normal(size=(8, 4))
    c = _cpu_cache(k, v, G=2, H=4, seg_lens=lens)
    d, lengths, ks, vs = akvc.parse_akvc(akvc.export_akvc(c, per_query_head=True))
    assert d == 4 and lengths == [3, 3, 5, 5]
    assert np.array_equal(ks[1], k[:3]) and np.array_equal(vs[2], v[3:8])
    d, lengths, ks, vs = akvc.parse_akvc(akvc.export_akvc(c, per_query_head=False))
    assert lengths == [3, 5] and np.array_equal(ks[1], k[3:8])
    with pytest.raises(OutOfRange):
        akvc.export_akvc(c, p=1)


def test_malformed_inputs_raise_format_error():
    good = akvc.export_akvc(_cpu_cache(np.ones((2, 2)), np.zeros((2, 2)), G=1, H=1, seg_lens=[2]))
    for bad in (good[:3], b"AKVX" + good[4:], good[:4] + struct.pack("<I", 2) + good[8:], good[:-1], good[:20]):
        with pytest.raises(FormatError):
            akvc.parse_akvc(bad)


@pytest.mark.gpu
def test_export_matches_oracle_evict_layer(dev, oracle_mod):
    import paper_2407_11550_b200 as A
    O = oracle_mod
    rng = np.random.default_rng(4)
    H, G, m, n, d, LB = 8, 2, 3, 40, 8, 30
    q = rng.normal(size=(H, m, d))
    ko, vo = rng.normal(size=(G, n, d)), rng.normal(size=(G, n, d))
    kw, vw = rng.normal(size=(G, m, d)), rng.normal(size=(G, m, d))
    K = np.concatenate([ko, kw], axis=1)
    V = np.concatenate([vo, vw], axis=1)
    T = lambda x: torch.as_tensor(np.ascontiguousarray(x)[None], device=dev)  # noqa: E731
    cache = A.compress(T(q), T(K), T(V), LB, kind="ada_snapkv", pool_kernel=3, alpha=0.2)
    r = O.evict_layer(q, ko, vo, kw, vw, LB, kind="ada_snapkv", pool_kernel=3, alpha=0.2)
    # reference layout: query head i holds group i // g's retained rows (policies.hpp:276)
    gs = H // G
    off = np.concatenate([[0], np.cumsum(r.ret_len)])
    heads_k = [torch.as_tensor(r.k_ret[off[i // gs]:off[i // gs + 1]]) for i in range(H)]
    heads_v = [torch.as_tensor(r.v_ret[off[i // gs]:off[i // gs + 1]]) for i in range(H)]
    assert akvc.export_akvc(cache) == akvc._flatten_bytes(heads_k, heads_v, d)
    # an imported file decodes like the original cache (one segment per stored head, g = 1)
    data = akvc.export_akvc(cache, per_query_head=False)
    back = akvc.import_akvc(data, dev, dtype=torch.float64)
    qg = torch.as_tensor(rng.normal(size=(1, G, d)), device=dev)
    o1 = A.decode(qg.repeat_interleave(H // G, dim=1), cache)  # every member head asks the same query
    o2 = A.decode(qg, back)
    for g in range(G):
        assert torch.allclose(o1[0, g * (H // G)], o2[0, g], rtol=1e-12, atol=1e-12)
    segs = [cache.segment(0, g) for g in range(G)]
    for g in range(G):
        kr, vr = back.segment(0, g)
        assert torch.equal(kr, segs[g][0]) and torch.equal(vr, segs[g][1])
