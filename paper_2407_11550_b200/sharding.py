"""Multi-GPU sharding of the compression path.

Batch sharding (configs 3, 5): requests are independent -- rank r takes requests r::N and
no collective touches the data path (`batch_shard`).

KV-group sharding (config 4: Llama-3.1-70B's 8 KV groups on 8 GPUs): scoring, per-group
selection, compaction and decode are group-local; the single cross-rank dependency is
Algorithm 1's layer-wide top-B (adaptive_allocation, budget.hpp:118-140).  Each rank takes
its local top-min(B, G_local*n_o) candidates with the same selection kernel, ONE all-gather
exchanges (score, global group, position) triples, and every rank runs the identical
deterministic merge: the union of the local top-B sets contains the global top-B, and
ordering the union by (global group, position) preserves the reference's (w desc, head asc,
pos asc) tie order, so the merged counts equal the single-GPU B* exactly.  The safeguard
blend and zero-budget repair (budget.hpp:145-158, policies.hpp:178-196) then run with the
TRUE capacities (n_o per group) on every rank, and each rank selects its own groups with the
resulting budgets.

The selection primitives are injected (`Selector`): `CudaSelector` calls the C ABI kernels;
the CPU tests substitute an oracle-backed selector to exercise exactly this orchestration
with gloo at world size 2.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Protocol, Sequence

import numpy as np
import torch
import torch.distributed as dist


def batch_shard(n_requests: int, rank: int, world: int) -> list[int]:
    """Requests owned by `rank` under batch sharding (weak scaling, no collective)."""
    return list(range(rank, n_requests, world))


class Selector(Protocol):
    def local_topk(self, scores: torch.Tensor, k: int) -> list[np.ndarray]:
        """scores [G_local, n_o]; per local group, the positions of its members of the
        layer-wide (over the local groups) top-k, ascending."""

    def union_counts(self, rows: Sequence[np.ndarray], total: int) -> np.ndarray:
        """Algorithm-1 counts of the top-`total` over ragged rows (flat order ties)."""

    def blend_repair(self, raw: np.ndarray, total: int, alpha: float, caps: np.ndarray) -> np.ndarray:
        """safeguard_blend with caps, then repair_zero_budgets."""

    def given_topk(self, scores: torch.Tensor, budgets: np.ndarray) -> list[np.ndarray]:
        """Per-group topk_decision with the given budgets; kept positions per group."""


class CudaSelector:
    """Selection on the device through the C ABI (paper_2407_11550_b200.ops)."""

    def __init__(self):
        from . import ops
        self.ops = ops

    def local_topk(self, scores, k):
        G, n = scores.shape
        off = np.arange(G + 1, dtype=np.int64) * n
        r = self.ops.segmented_select(scores.reshape(1, G * n).float().contiguous(), off, int(k), "adaptive",
                                      want_keep=False, want_pos=True)
        counts = r["budgets"][0].cpu().numpy()
        pos = r["kept_pos"][0].cpu().numpy()
        out, c0 = [], 0
        for c in counts:
            out.append(pos[c0:c0 + c].astype(np.int64))
            c0 += c
        return out

    def union_counts(self, rows, total):
        lens = [len(r) for r in rows]
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        flat = np.concatenate(rows).astype(np.float32) if sum(lens) else np.zeros(1, np.float32)
        dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(flat, device=dev).reshape(1, -1)
        if int(off[-1]) == 0:
            return np.zeros(len(rows), np.int64)
        r = self.ops.segmented_select(t, off, int(total), "adaptive", want_keep=False, want_pos=False)
        return r["budgets"][0].cpu().numpy().astype(np.int64)

    def blend_repair(self, raw, total, alpha, caps):
        b = self.ops.safeguard_blend(raw, total, len(raw), alpha, caps)
        return self.ops.repair_zero_budgets(b, caps)

    def given_topk(self, scores, budgets):
        G, n = scores.shape
        off = np.arange(G + 1, dtype=np.int64) * n
        bud = torch.as_tensor(np.asarray(budgets, np.int32)[None, :], device=scores.device)
        r = self.ops.segmented_select(scores.reshape(1, G * n).float().contiguous(), off, 0, "given", budgets=bud,
                                      want_keep=False, want_pos=True)
        pos = r["kept_pos"][0].cpu().numpy()
        out, c0 = [], 0
        for c in budgets:
            out.append(pos[c0:c0 + int(c)].astype(np.int64))
            c0 += int(c)
        return out


@dataclass
class ShardedAllocation:
    raw: np.ndarray        # [G] Algorithm-1 counts B* (identical on every rank)
    budgets: np.ndarray    # [G] after safeguard + repair (identical on every rank)
    kept: list             # local groups: kept positions (ascending), per group
    candidates: int        # candidates contributed by this rank


def _f32_bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32).view(np.int32).astype(np.int64)


def _bits_f32(b: np.ndarray) -> np.ndarray:
    return b.astype(np.int32).view(np.float32)


def kv_group_sharded_allocation(local_scores: torch.Tensor, g0: int, G: int, total: int, alpha: float,
                                selector: Selector, group=None, blend: bool = True) -> ShardedAllocation:
    """Layer-wide adaptive allocation over KV groups sharded across ranks.

    local_scores [G_local, n_o] (this rank's groups g0 .. g0+G_local-1, fp32 scores);
    total = outside budget of the layer (layer_budget - m*G).  One all-gather.
    """
    G_local, n_o = local_scores.shape
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    # 1) local top-k candidates (same kernel as the single-GPU path)
    k_local = min(int(total), G_local * n_o)
    pos = selector.local_topk(local_scores, k_local) if k_local > 0 else [np.zeros(0, np.int64)] * G_local
    sc = local_scores.detach().float().cpu().numpy()
    trip = [np.stack([_f32_bits(sc[gl][p]), np.full(len(p), g0 + gl, np.int64), p], axis=1)
            for gl, p in enumerate(pos) if len(p)]
    cand = np.concatenate(trip) if trip else np.zeros((0, 3), np.int64)
    # 2) one all-gather of (score bits, global group, position), padded to a common length
    n_mine = torch.tensor([cand.shape[0]], dtype=torch.int64)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dev = local_scores.device if dist.is_initialized() and dist.get_backend(group) == "nccl" else torch.device("cpu")
    if world > 1:
        if dev.type == "cuda":
            n_mine = n_mine.to(dev)
            counts = [c.to(dev) for c in counts]
        dist.all_gather(counts, n_mine, group=group)
    else:
        counts = [n_mine]
    kmax = max(int(c.item()) for c in counts)
    buf = np.full((max(kmax, 1), 3), -1, np.int64)
    buf[:cand.shape[0]] = cand
    mine = torch.as_tensor(buf, device=dev)
    if world > 1:
        gathered = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine, group=group)
        allc = np.concatenate([g.cpu().numpy()[:int(c.item())] for g, c in zip(gathered, counts)])
    else:
        allc = cand
    # 3) deterministic merge: union ordered by (global group, position) = the reference's flat order
    rows = []
    for g in range(G):
        sel = allc[allc[:, 1] == g]
        sel = sel[np.argsort(sel[:, 2], kind="stable")]
        rows.append(_bits_f32(sel[:, 0]).astype(np.float64) if len(sel) else np.zeros(0))
    raw = selector.union_counts(rows, int(total))
    caps = np.full(G, n_o, np.int64)
    budgets = selector.blend_repair(raw, int(total), float(alpha), caps) if blend else raw
    # 4) this rank's groups with their budgets
    kept = selector.given_topk(local_scores, budgets[g0:g0 + G_local])
    return ShardedAllocation(raw=np.asarray(raw), budgets=np.asarray(budgets), kept=kept,
                             candidates=int(cand.shape[0]))


def pack_candidate_bytes(k: int) -> int:
    """Bytes one rank contributes to the all-gather for k candidates (3 x int64 each)."""
    return k * 3 * struct.calcsize("q")
