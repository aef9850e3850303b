"""Regenerate the committed golden fixtures from the UNMODIFIED reference.

Runs only in the build container (needs /root/reference to build
oracle/_ref/).  The outputs are small .npz files committed under tests/golden/
so that the GPU box -- where /root/reference does not exist -- can check the
CUDA path and the C restatement against the reference's own results.

    python tests/golden/make_golden.py

Fixtures:
  config1.npz      reference trace generator (trace.hpp:277-350), Llama-shaped
                   layer h=32, gqa 4, n=4064, d_h=128, window 32, seed 7,
                   ada_snapkv alpha=0.2 pool 7, layer_budget 8192
                   (BASELINE.json configs[0]).  Group scores f64 + the
                   reference's allocation and decision: the "identical scores
                   => bit-exact budgets/indices" gate.
  demo.npz         same generator at the worked-example shape
                   (demo/worked_example.cpp:37-45): h=4, n=256, d_h=8, m=8.
  evict_small.npz  seeded random evict_layer instances (all five kinds) with the
                   reference's full outputs, including retained K/V rows.
  select_ties.npz  adversarial selection inputs (all-equal, quantised k/64,
                   underflowed zeros) with the reference's adaptive_allocation,
                   safeguard_blend and topk_decision results.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def run_generator(name, h, gqa, n, d_h, window, seed, budget, kind, alpha, pool):
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "golden"], check=True)
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_golden")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([exe, td, name, str(h), str(gqa), str(n), str(d_h), str(window), str(seed),
                        str(budget), kind, repr(alpha), str(pool)], check=True)
        G = h // gqa
        scores = np.fromfile(os.path.join(td, f"{name}.scores.f64"), np.float64).reshape(G, n)
        alloc = np.fromfile(os.path.join(td, f"{name}.alloc.i64"), np.int64)
        keep = np.fromfile(os.path.join(td, f"{name}.keep.u8"), np.uint8).reshape(G, n)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), scores=scores, alloc=alloc, keep=keep,
                        meta=np.array([h, gqa, n, d_h, window, seed, budget], np.int64),
                        kind=np.array(kind), alpha=np.array(alpha), pool=np.array(pool))
    print(name, "alloc", "|".join(map(str, alloc)))


def evict_small():
    rng = np.random.default_rng(20241018)
    cases = {}
    idx = 0
    for trial in range(12):
        G = int(rng.integers(1, 4))
        g = int(rng.integers(1, 5))
        H = G * g
        m = int(rng.integers(1, 5))
        n = int(rng.integers(8, 48))
        d = int(rng.choice([1, 2, 3, 4, 8, 16]))
        q = rng.normal(size=(H, m, d))
        ko, vo = rng.normal(size=(G, n, d)), rng.normal(size=(G, n, d))
        kw, vw = rng.normal(size=(G, m, d)), rng.normal(size=(G, m, d))
        LB = m * G + G + int(rng.integers(0, G * (n - 1) + 1))
        pk = int(rng.choice([1, 3, 5, 7]))
        alpha = float(rng.random())
        for kind in O.KINDS:
            r = O.evict_layer(q, ko, vo, kw, vw, LB, kind=kind, pool_kernel=pk, alpha=alpha, impl="ref")
            p = f"c{idx}_"
            cases.update({p + "q": q, p + "k_out": ko, p + "v_out": vo, p + "k_win": kw, p + "v_win": vw,
                          p + "params": np.array([LB, pk, O.KINDS[kind]], np.int64),
                          p + "alpha": np.array(alpha),
                          p + "group_scores": r.group_scores, p + "alloc": r.alloc, p + "keep": r.keep,
                          p + "k_ret": r.k_ret, p + "v_ret": r.v_ret, p + "ret_len": r.ret_len})
            idx += 1
    cases["count"] = np.array(idx)
    np.savez_compressed(os.path.join(OUT, "evict_small.npz"), **cases)
    print("evict_small", idx, "cases")


def select_ties():
    rng = np.random.default_rng(7)
    G, n = 8, 300
    dists = {
        "equal": np.full((G, n), 0.25),
        "quantised": np.floor(rng.random((G, n)) * 64) / 64.0,
        "underflow": np.where(rng.random((G, n)) < 0.7, 0.0, rng.random((G, n)) * 1e-3),
        "random": rng.exponential(size=(G, n)),
    }
    out = {}
    for name, s in dists.items():
        for k in (0, 1, 17, 400, 1203, G * n):
            raw = O.adaptive_allocation(list(s), k, impl="ref")
            out[f"{name}_{k}_raw"] = raw
            caps = np.full(G, n, np.int64)
            for alpha in (0.0, 0.2, 1.0):
                out[f"{name}_{k}_{alpha}_blend"] = O.safeguard_blend(raw, k, G, alpha, caps, impl="ref")
        out[f"{name}_scores"] = s
        ks = rng.integers(0, n + 1, size=G)
        out[f"{name}_topk_k"] = ks
        out[f"{name}_topk_keep"] = np.stack([O.topk_decision(s[i], int(ks[i]), impl="ref") for i in range(G)])
    np.savez_compressed(os.path.join(OUT, "select_ties.npz"), **out)
    print("select_ties", len(dists), "distributions")


if __name__ == "__main__":
    run_generator("config1", 32, 4, 4064, 128, 32, 7, 8192, "ada_snapkv", 0.2, 7)
    run_generator("demo", 4, 1, 256, 8, 8, 7, (256 + 8) * 4 // 4, "ada_snapkv", 0.2, 7)
    evict_small()
    select_ties()
