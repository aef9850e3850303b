"""Multi-GPU sharding of the compression path.

Batch sharding (configs 3, 5): requests are independent -- rank r takes requests r::N and
no collective touches the data path (`batch_shard`).

KV-group sharding (config 4: Llama-3.1-70B's 8 KV groups over the GPUs): scoring, per-group
selection, compaction and decode are group-local; the single cross-rank dependency is
Algorithm 1's layer-wide top-B (adaptive_allocation, budget.hpp:118-140).  Every rank
  1. takes its local top-k_local candidates, k_local = min(B, G_local * n_o), with the same
     selection kernel (segment-major, positions ascending: the reference's flat order);
  2. contributes ONE fixed-size int32 payload [G_local counts | k_local score bits | k_local
     positions] to ONE all-gather (k_local is known a priori, so there is no count exchange);
  3. scatters the gathered candidates into a [G, S] union (S = min(k_local, n_o) slots per
     group, empty slots = -1, below every score) ordered by (group, position) and runs the
     adaptive selection + safeguard_blend + repair_zero_budgets over it on the device.
The union of the local top-B sets contains the global top-B and keeps the (w desc, head asc,
pos asc) tie order, so the merged counts equal the single-GPU B* bit for bit; segment size S
equals the true capacity n_o whenever a cap can bind (budget.hpp:145-158), so the blended and
repaired budgets do too.  4. Each rank then selects its own groups with those budgets.
Nothing leaves the device on the CUDA path (no .cpu(), no numpy).

The selection primitives are injected (`Selector`): `CudaSelector` calls the C ABI kernels;
the CPU tests substitute an oracle-backed selector to run exactly this orchestration with
gloo at world size 2.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol

import numpy as np
import torch
import torch.distributed as dist


def batch_shard(n_requests: int, rank: int, world: int) -> list[int]:
    """Requests owned by `rank` under batch sharding (weak scaling, no collective)."""
    return list(range(rank, n_requests, world))


class Selector(Protocol):
    def topk(self, scores: torch.Tensor, k: int) -> tuple[torch.Tensor, torch.Tensor]:
        """scores [S, n] fp32: the layer-wide top-k over the S segments (Algorithm 1, flat-order
        ties) -> (counts int32 [S], kept positions int32 [k], segment-major, ascending)."""

    def allocate(self, union: torch.Tensor, total: int, alpha: float, blend: bool) -> tuple[torch.Tensor,
                                                                                              torch.Tensor]:
        """union [G, S] fp32 -> (raw Algorithm-1 counts, budgets after safeguard_blend with caps
        S and repair_zero_budgets), both int32 [G]."""

    def given(self, scores: torch.Tensor, budgets: torch.Tensor) -> torch.Tensor:
        """Per-segment topk_decision with the given budgets -> kept positions int32
        [sum(budgets)], segment-major, ascending."""


class CudaSelector:
    """Selection on the device through the C ABI (paper_2407_11550_b200.ops)."""

    def __init__(self):
        from . import ops
        self.ops = ops

    def topk(self, scores, k):
        S, n = scores.shape
        off = np.arange(S + 1, dtype=np.int64) * n
        r = self.ops.segmented_select(scores.reshape(1, S * n).float().contiguous(), off, int(k), "adaptive",
                                      want_keep=False, want_pos=True)
        return r["budgets"][0].clone(), r["kept_pos"][0, :k].clone()

    def allocate(self, union, total, alpha, blend):
        G, S = union.shape
        off = np.arange(G + 1, dtype=np.int64) * S
        r = self.ops.segmented_select(union.reshape(1, G * S).contiguous(), off, int(total), "adaptive",
                                      blend=blend, alpha=alpha, repair=blend, want_keep=False, want_pos=False,
                                      want_raw=True)
        return r["raw"][0].clone(), r["budgets"][0].clone()

    def given(self, scores, budgets):
        S, n = scores.shape
        off = np.arange(S + 1, dtype=np.int64) * n
        r = self.ops.segmented_select(scores.reshape(1, S * n).float().contiguous(), off, 0, "given",
                                      budgets=budgets.reshape(1, S).to(torch.int32).contiguous(), want_keep=False,
                                      want_pos=True)
        return r["kept_pos"][0]


@dataclass
class ShardedAllocation:
    raw: torch.Tensor       # int32 [G] Algorithm-1 counts B* (identical on every rank)
    budgets: torch.Tensor   # int32 [G] after safeguard + repair (identical on every rank)
    kept_pos: torch.Tensor  # int32: this rank's groups' kept positions, group-major, ascending
    candidates: int         # candidates contributed by this rank (k_local)
    payload_bytes: int      # bytes this rank sends through the one all-gather

    def kept(self, g0: int, G_local: int) -> list:
        """Per local group kept positions (host lists; for checks, not the data path)."""
        b = self.budgets[g0:g0 + G_local].cpu().tolist()
        kp = self.kept_pos.cpu()
        out, c = [], 0
        for n in b:
            out.append(kp[c:c + n])
            c += n
        return out


def kv_group_sharded_allocation(local_scores: torch.Tensor, g0: int, G: int, total: int, alpha: float,
                                selector: Selector, group=None, blend: bool = True) -> ShardedAllocation:
    """Layer-wide adaptive allocation over KV groups sharded across ranks (one all-gather).

    local_scores [G_local, n_o] fp32: this rank's groups g0 .. g0 + G_local - 1 (every rank
    holds the same number of groups); total = outside budget of the layer (layer_budget - m G).
    """
    G_local, n_o = local_scores.shape
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if G_local * world != G:
        raise ValueError("kv_group_sharded_allocation: every rank must hold G / world groups")
    dev = local_scores.device
    # 1) local top-k candidates (same kernel as the single-GPU path)
    k_local = min(int(total), G_local * n_o)
    counts, pos = selector.topk(local_scores, k_local)
    # 2) one all-gather of a fixed-size payload: [counts | score bits | positions]
    payload = (_cuda_pack if local_scores.is_cuda else _torch_pack)(local_scores, counts, pos, k_local)
    if dist.is_initialized():  # (also at world size 1: the same NCCL path the ranks take)
        if dist.get_backend(group) == "nccl":
            gathered = torch.empty((world, payload.numel()), dtype=torch.int32, device=dev)
            dist.all_gather_into_tensor(gathered, payload, group=group)
        else:  # gloo (CPU tests): the same single exchange as a list all-gather
            parts = [torch.empty_like(payload) for _ in range(world)]
            dist.all_gather(parts, payload, group=group)
            gathered = torch.stack(parts)
    else:
        gathered = payload.reshape(1, -1)
    # 3) union [G, S] ordered by (group, position); empty slots -1 (below every score >= 0)
    S = max(1, min(k_local, n_o))
    union = (_cuda_union if gathered.is_cuda else _torch_union)(gathered, world, G_local, k_local, S)
    raw, budgets = selector.allocate(union.float(), int(total), float(alpha), blend)
    # 4) this rank's groups with the merged budgets
    kept_pos = selector.given(local_scores, budgets[g0:g0 + G_local])
    return ShardedAllocation(raw=raw, budgets=budgets, kept_pos=kept_pos, candidates=k_local,
                             payload_bytes=int(payload.numel()) * 4)


def compress_kv_group_sharded(q, k, v, layer_budget: int, G: int, *, g0: int, group=None, alpha=0.2,
                              pool_kernel=7, reserve=0, selector: Selector | None = None):
    """evict_layer (policies.hpp:204-293) for ONE problem whose G KV groups are sharded over the
    ranks: q [H_local, m, d], k, v [G_local, n, d] hold this rank's groups g0 .. g0 + G_local - 1
    (and their g * G_local query heads).  Scores, the local top-k, the per-group selection and
    the compaction are local; the layer-wide allocation is kv_group_sharded_allocation.
    Returns (CompressedCache over the local groups, ShardedAllocation)."""
    from . import ops
    from . import _lib as L
    import ctypes as C
    H_l, m, d = q.shape
    G_l, n, _ = k.shape
    n_o = n - m
    scores = ops.window_scores(q[None], k[None], pool_kernel)[0]            # [G_local, n_o]
    alloc = kv_group_sharded_allocation(scores, g0, G, int(layer_budget) - m * G, alpha,
                                        selector or CudaSelector(), group=group)
    bud_l = alloc.budgets[g0:g0 + G_l].contiguous()
    dev = q.device
    # local planes sized by the bound on the local groups' share (no host read of the budgets):
    # at most min(B, G_local n_o) outside rows plus the window (and reserve) rows
    lb_l = min(int(layer_budget) - m * G, G_l * n_o) + m * G_l
    rows = lb_l + G_l * reserve
    out = ops.CompressedCache(k=torch.empty((max(rows, 1), d), dtype=k.dtype, device=dev),
                              v=torch.empty((max(rows, 1), d), dtype=k.dtype, device=dev),
                              seg_start=torch.empty(G_l, dtype=torch.int32, device=dev),
                              seqlens=torch.empty(G_l, dtype=torch.int32, device=dev),
                              seg_cap=torch.empty(G_l, dtype=torch.int32, device=dev),
                              budgets=bud_l.to(torch.int32), P=1, H=H_l, G=G_l, m=m, d=d, reserve=reserve,
                              layer_budget=lb_l)
    shape = ops.layer_shape(1, H_l, G_l, m, n_o, d)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    L.check(L.lib().adakv_gather(ops._dt(k), C.byref(shape), lb_l, None, p(k), p(v), p(out.budgets),
                                 p(alloc.kept_pos), max(int(alloc.kept_pos.numel()), 1), int(reserve), p(out.k),
                                 p(out.v), p(out.seg_start), p(out.seqlens), p(out.seg_cap), None, ops._stream()))
    return out, alloc


def _torch_pack(local_scores, counts, pos, k):
    """The all-gather payload [counts | candidate score bits | positions] with torch ops (CPU path)."""
    G_local, n_o = local_scores.shape
    dev = local_scores.device
    flat = local_scores.reshape(-1).float()
    gidx = torch.repeat_interleave(torch.arange(G_local, device=dev), counts.to(torch.int64),
                                   output_size=k) if k else torch.zeros(0, dtype=torch.int64, device=dev)
    cand = flat[gidx * n_o + pos.to(torch.int64)]
    return torch.cat([counts.to(torch.int32), cand.view(torch.int32), pos.to(torch.int32)])


def _torch_union(gathered, world, G_local, k, S):
    """The [world G_local, S] candidate union with torch ops (CPU path)."""
    dev = gathered.device
    G = world * G_local
    g_counts = gathered[:, :G_local].reshape(-1).to(torch.int64)                 # [G] (rank-major = group order)
    g_scores = gathered[:, G_local:G_local + k].contiguous().view(torch.float32)  # [world, k]
    g_start = (torch.cumsum(g_counts.view(world, G_local), 1) - g_counts.view(world, G_local)).reshape(-1)
    j = torch.arange(S, device=dev)
    valid = j[None, :] < g_counts[:, None]                                        # [G, S]
    src = (g_start[:, None] + j[None, :]).clamp(max=max(k - 1, 0))                # index within the rank's list
    rank_of = torch.arange(G, device=dev) // G_local
    return torch.where(valid, g_scores[rank_of[:, None], src], torch.full((), -1.0, device=dev))


def _cuda_pack(local_scores, counts, pos, k):
    """adakv_shard_pack_candidates: the all-gather payload in one kernel."""
    import ctypes as C
    from . import _lib as L
    from . import ops
    G_local, n_o = local_scores.shape
    sc = local_scores.float().contiguous()
    cnt = counts.to(torch.int32).contiguous()
    ps = pos.to(torch.int32).contiguous()
    payload = torch.empty(G_local + 2 * k, dtype=torch.int32, device=local_scores.device)
    L.check(L.lib().adakv_shard_pack_candidates(C.c_void_p(sc.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                                C.c_void_p(ps.data_ptr()) if k else None, G_local, n_o, k,
                                                C.c_void_p(payload.data_ptr()), ops._stream()))
    return payload


def _cuda_union(gathered, world, G_local, k, S):
    """adakv_shard_build_union: the [G, S] candidate union in one kernel."""
    import ctypes as C
    from . import _lib as L
    from . import ops
    g = gathered.to(torch.int32).contiguous()
    union = torch.empty((world * G_local, S), dtype=torch.float32, device=gathered.device)
    L.check(L.lib().adakv_shard_build_union(C.c_void_p(g.data_ptr()), world, G_local, k, S,
                                            C.c_void_p(union.data_ptr()), ops._stream()))
    return union


def pack_candidate_bytes(k: int, G_local: int) -> int:
    """Bytes one rank contributes to the all-gather: G_local counts + k score bits + k positions."""
    return 4 * (G_local + 2 * k)
