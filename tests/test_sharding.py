"""Multi-process (gloo, world size 2, CPU) tests of the sharded compression path.

KV-group sharding must reproduce the single-process allocation bit-exactly: the union of
per-rank local top-B candidates exchanged by ONE all-gather, merged in (group, position)
order, gives the reference's Algorithm-1 counts (budget.hpp:118-140) even under heavy ties.
The selection primitives are the oracle's here (no GPU on this box); on the GPU the same
orchestration runs with CudaSelector + NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_11550_b200.sharding import batch_shard, kv_group_sharded_allocation


class OracleSelector:
    def __init__(self):
        from oracle import oracle as O
        self.O = O

    def local_topk(self, scores, k):
        rows = [r.astype(np.float64) for r in scores.float().numpy()]
        raw = self.O.adaptive_allocation(rows, k)
        return [np.nonzero(self.O.topk_decision(rows[g], int(raw[g])))[0] for g in range(len(rows))]

    def union_counts(self, rows, total):
        return self.O.adaptive_allocation(list(rows), total)

    def blend_repair(self, raw, total, alpha, caps):
        b = self.O.safeguard_blend(raw, total, len(raw), alpha, caps)
        return self.O.repair_zero_budgets(b, caps)

    def given_topk(self, scores, budgets):
        rows = [r.astype(np.float64) for r in scores.float().numpy()]
        return [np.nonzero(self.O.topk_decision(rows[g], int(budgets[g])))[0] for g in range(len(rows))]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scores(seed, G, n, kind):
    rng = np.random.default_rng(seed)
    if kind == "ties":
        return (np.floor(rng.random((G, n)) * 16) / 16).astype(np.float32)
    if kind == "equal":
        return np.full((G, n), 0.125, np.float32)
    return rng.exponential(size=(G, n)).astype(np.float32)


def _worker(rank, world, port, cases, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sel = OracleSelector()
    res = []
    for (seed, G, n, total, alpha, kind) in cases:
        s = _scores(seed, G, n, kind)
        gl = G // world
        local = torch.as_tensor(s[rank * gl:(rank + 1) * gl])
        r = kv_group_sharded_allocation(local, rank * gl, G, total, alpha, sel)
        res.append((r.raw.tolist(), r.budgets.tolist(), [k.tolist() for k in r.kept]))
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


CASES = [(1, 8, 300, 1200, 0.2, "random"), (2, 8, 300, 1200, 0.2, "ties"), (3, 4, 100, 50, 0.2, "equal"),
         (4, 8, 64, 8 * 64, 0.5, "random"), (5, 2, 500, 3, 1.0, "ties"), (6, 8, 200, 8, 0.2, "random")]


def test_kv_group_sharded_matches_single_process(oracle_mod):
    O = oracle_mod
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (seed, G, n, total, alpha, kind) in enumerate(CASES):
        s = _scores(seed, G, n, kind).astype(np.float64)
        raw = O.adaptive_allocation(list(s), total)
        b = O.repair_zero_budgets(O.safeguard_blend(raw, total, G, alpha, np.full(G, n)), np.full(G, n))
        keep = [np.nonzero(O.topk_decision(s[g], int(b[g])))[0].tolist() for g in range(G)]
        gl = G // world
        for rank in range(world):
            r_raw, r_b, r_kept = results[rank][ci]
            assert r_raw == raw.tolist(), (ci, rank)
            assert r_b == b.tolist(), (ci, rank)
            assert r_kept == keep[rank * gl:(rank + 1) * gl], (ci, rank)


def test_batch_shard_partitions_requests():
    for n in (1, 7, 32):
        for w in (1, 2, 4, 8):
            parts = [batch_shard(n, r, w) for r in range(w)]
            assert sorted(sum(parts, [])) == list(range(n))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


@pytest.mark.gpu
def test_kv_group_sharded_cuda_selector_single_rank(dev, oracle_mod):
    """World size 1 with the CUDA selector: the merge path reproduces the single-GPU budgets."""
    from paper_2407_11550_b200.sharding import CudaSelector
    O = oracle_mod
    G, n, total = 8, 500, 1000
    s = _scores(9, G, n, "ties")
    r = kv_group_sharded_allocation(torch.as_tensor(s, device=dev), 0, G, total, 0.2, CudaSelector())
    s64 = s.astype(np.float64)
    raw = O.adaptive_allocation(list(s64), total)
    b = O.repair_zero_budgets(O.safeguard_blend(raw, total, G, 0.2, np.full(G, n)), np.full(G, n))
    assert r.raw.tolist() == raw.tolist() and r.budgets.tolist() == b.tolist()
    for g in range(G):
        assert r.kept[g].tolist() == np.nonzero(O.topk_decision(s64[g], int(b[g])))[0].tolist()
