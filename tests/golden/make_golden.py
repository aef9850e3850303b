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
  fig3_dump.npz    the reference's run_comparison (report.hpp:161-345) on a small
                   trace of its own generator (h=8, n=256, d_h=4, 6 samples, seed 5):
                   every sample's inputs (K/V, window queries, decode query, W_o) and
                   the reference's rows (loss, epsilon, epsilon*, epsilon**, retained
                   mass, allocation) for ada_snapkv / snapkv at fractions 0.2 / 0.4.
  fig3_accept.npz  acceptance check #7 (acceptance_test.cpp:134-163) as the reference
                   runs it: 200 samples, fractions 0.2 / 0.4 -- per-sample losses of
                   both policies and the win fractions.
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


def _parse_rows(path):
    rows, aggs = [], []
    for line in open(path):
        t = line.split()
        if t[0] == "agg":
            aggs.append([float(t[1]), int(t[2]), int(t[3]), float(t[4])])
        else:
            rows.append((int(t[0]), float(t[1]), t[2], int(t[3]), [float(x) for x in t[4:9]],
                         [int(x) for x in t[9:]]))
    return rows, np.array(aggs)


def fig3():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "fig3"], check=True)
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_fig3")
    h, n, d, m, S, D = 8, 256, 4, 32, 6, (8 + 8) * 4
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([exe, "dump", td], check=True)
        wo = np.fromfile(os.path.join(td, "wo.f64"), np.float64).reshape(h, d, D)
        arrs = {k: [] for k in ("k_out", "v_out", "k_win", "v_win", "q_win", "q_dec")}
        for si in range(S):
            x = np.fromfile(os.path.join(td, f"s{si}.f64"), np.float64)
            o = 0
            for key, shape in (("k_out", (h, n, d)), ("v_out", (h, n, d)), ("k_win", (h, m, d)),
                               ("v_win", (h, m, d)), ("q_win", (h, m, d)), ("q_dec", (h, d))):
                cnt = int(np.prod(shape))
                arrs[key].append(x[o:o + cnt].reshape(shape))
                o += cnt
            assert o == x.size
        rows, aggs = _parse_rows(os.path.join(td, "rows.txt"))
    out = {k: np.stack(v) for k, v in arrs.items()}
    out["wo"] = wo
    out["row_sample"] = np.array([r[0] for r in rows], np.int64)
    out["row_fraction"] = np.array([r[1] for r in rows])
    out["row_policy"] = np.array([r[2] for r in rows])
    out["row_budget"] = np.array([r[3] for r in rows], np.int64)
    out["row_values"] = np.array([r[4] for r in rows])      # loss, epsilon, eps*, eps**, mass
    out["row_alloc"] = np.array([r[5] for r in rows], np.int64)
    out["aggregates"] = aggs
    np.savez_compressed(os.path.join(OUT, "fig3_dump.npz"), **out)
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([exe, "accept", os.path.join(td, "a.txt")], check=True)
        rows, aggs = _parse_rows(os.path.join(td, "a.txt"))
    np.savez_compressed(os.path.join(OUT, "fig3_accept.npz"),
                        sample=np.array([r[0] for r in rows], np.int64),
                        fraction=np.array([r[1] for r in rows]), policy=np.array([r[2] for r in rows]),
                        loss=np.array([r[4][0] for r in rows]), aggregates=aggs)
    print("fig3: dump rows", len(out["row_sample"]), "accept win fractions", aggs[:, 3].tolist())


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "fig3":
        fig3()
        sys.exit(0)
    run_generator("config1", 32, 4, 4064, 128, 32, 7, 8192, "ada_snapkv", 0.2, 7)
    run_generator("demo", 4, 1, 256, 8, 8, 7, (256 + 8) * 4 // 4, "ada_snapkv", 0.2, 7)
    evict_small()
    select_ties()
    fig3()
