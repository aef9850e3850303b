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
    """The same three primitives as CudaSelector, computed by the C oracle on the host."""

    def __init__(self):
        from oracle import oracle as O
        self.O = O

    def topk(self, scores, k):
        rows = [r.astype(np.float64) for r in scores.float().numpy()]
        raw = self.O.adaptive_allocation(rows, k)
        pos = [np.nonzero(self.O.topk_decision(rows[g], int(raw[g])))[0] for g in range(len(rows))]
        return torch.as_tensor(raw, dtype=torch.int32), torch.as_tensor(np.concatenate(pos), dtype=torch.int32)

    def allocate(self, union, total, alpha, blend):
        rows = [r.astype(np.float64) for r in union.float().numpy()]
        raw = self.O.adaptive_allocation(rows, total)
        caps = np.full(len(rows), union.shape[1], np.int64)
        b = self.O.repair_zero_budgets(self.O.safeguard_blend(raw, total, len(raw), alpha, caps), caps) if blend else raw
        return torch.as_tensor(raw, dtype=torch.int32), torch.as_tensor(b, dtype=torch.int32)

    def given(self, scores, budgets):
        rows = [r.astype(np.float64) for r in scores.float().numpy()]
        pos = [np.nonzero(self.O.topk_decision(rows[g], int(budgets[g])))[0] for g in range(len(rows))]
        return torch.as_tensor(np.concatenate(pos), dtype=torch.int32)


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
        res.append((r.raw.tolist(), r.budgets.tolist(), [k.tolist() for k in r.kept(rank * gl, gl)],
                    r.payload_bytes))
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
            r_raw, r_b, r_kept, nbytes = results[rank][ci]
            assert nbytes == 4 * (gl + 2 * min(total, gl * n))  # one fixed-size payload per rank
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
    kept = r.kept(0, G)
    for g in range(G):
        assert kept[g].tolist() == np.nonzero(O.topk_decision(s64[g], int(b[g])))[0].tolist()


@pytest.mark.gpu
def test_kv_group_sharded_compress_nccl_world1(dev, oracle_mod, capfd):
    """The KV-group-sharded compress through a real NCCL communicator (world size 1 on this
    one-GPU box: the all-gather runs through NCCL) equals the single-GPU compress: budgets,
    segment layout and every retained row bit for bit (Llama-3.1-70B shapes, g = 8, 8K prompt)."""
    import paper_2407_11550_b200 as A
    from paper_2407_11550_b200.sharding import compress_kv_group_sharded
    from paper_2407_11550_b200.synthetic import planted_layer
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    os.environ["NCCL_DEBUG"] = "INFO"
    created = not dist.is_initialized()
    if created:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        H, G, m, n_o, d = 64, 8, 32, 8160, 128
        q, k, v = planted_layer(1, H, G, n_o, m, d, seed=44, dtype=torch.bfloat16, device=dev)
        LB = 512 * G
        ref = A.compress(q, k, v, LB, reserve=3)
        sh, alloc = compress_kv_group_sharded(q[0], k[0], v[0], LB, G, g0=0, reserve=3)
        torch.cuda.synchronize()
        assert alloc.budgets.cpu().tolist() == ref.budgets.cpu().tolist()
        assert alloc.payload_bytes == 4 * (G + 2 * (LB - m * G))
        for g in range(G):
            a, b = sh.segment(0, g), ref.segment(0, g)
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), g
        assert sh.seg_cap.cpu().tolist() == ref.seg_cap.cpu().tolist()
    finally:
        if created:
            dist.destroy_process_group()
    err = capfd.readouterr()
    print("\n".join(l for l in (err.out + err.err).splitlines() if "NCCL INFO" in l and ("comm" in l or "Init" in l))[:2000])


@pytest.mark.gpu
def test_shard_glue_kernels_match_torch_glue(dev):
    """adakv_shard_pack_candidates / adakv_shard_build_union (the sharded path's device glue)
    equal the torch formulation the CPU tests run, for three ranks' payloads with ragged
    per-group counts (including empty groups) and heavy ties."""
    from paper_2407_11550_b200.sharding import CudaSelector, _cuda_pack, _cuda_union, _torch_pack, _torch_union
    sel = CudaSelector()
    G_local, n_o, k, world = 2, 300, 250, 3
    payloads = []
    for r in range(world):
        s = torch.as_tensor(_scores(30 + r, G_local, n_o, "ties"), device=dev)
        if r == 1:
            s[1] = 0.0  # one group with no candidate above the others
        counts, pos = sel.topk(s, k)
        pc = _cuda_pack(s, counts, pos, k)
        pt = _torch_pack(s.cpu(), counts.cpu(), pos.cpu(), k)
        assert torch.equal(pc.cpu(), pt), r
        payloads.append(pc)
    gathered = torch.stack(payloads)
    S = min(k, n_o)
    uc = _cuda_union(gathered, world, G_local, k, S)
    ut = _torch_union(gathered.cpu(), world, G_local, k, S)
    assert torch.equal(uc.cpu().view(torch.int32), ut.view(torch.int32))
