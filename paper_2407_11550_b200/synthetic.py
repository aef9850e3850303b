"""Synthetic prompt caches with planted attention structure (bench + parity inputs).

Follows the reference generator's construction (trace.hpp:117-151 planted rows,
230-261 make_embeddings) applied directly in head space, as SURVEY.md §8(d)
prescribes for configs 2-5: per KV group a planted distribution p over the n_o
outside positions -- "sparse" (5% of positions in `runs` contiguous runs carry
`top_mass`, exponential tail) or "dispersed" (softmax of temp * N(0,1)) -- and a
unit direction u; outside keys K_j = (ln p_j + ln n_o) u + 0.05 eps, window keys
0.1 eps, window queries sqrt(d) u + 0.15 eps, values N(0, 1).  So
softmax(q.k/sqrt(d)) lands near p and the heads have realistic (non-uniform,
differently concentrated) score profiles.  Generated on the target device.
"""
from __future__ import annotations

import math

import torch


def planted_rows(G: int, n: int, gen: torch.Generator, frac_sparse=0.75, top_mass=0.95, temp=0.3,
                 runs=2, device="cpu") -> torch.Tensor:
    """[G, n] float32 planted probability rows (trace.hpp:117-171)."""
    rows = torch.empty((G, n), dtype=torch.float32, device=device)
    n_sparse = int(round(frac_sparse * G))
    order = torch.randperm(G, generator=gen, device="cpu").tolist()
    sparse = set(order[:n_sparse])
    s_cnt = math.ceil(0.05 * n)
    nruns = max(1, min(runs, s_cnt))
    for gi in range(G):
        if gi in sparse:
            spike = torch.zeros(n, dtype=torch.bool, device=device)
            for r in range(nruns):
                ln = s_cnt // nruns + (1 if r < s_cnt % nruns else 0)
                lo, hi = r * n // nruns, (r + 1) * n // nruns
                ln = min(ln, hi - lo)
                start = lo + int(torch.randint(0, hi - lo - ln + 1, (1,), generator=gen).item())
                spike[start:start + ln] = True
            u = torch.rand(n, generator=gen, device="cpu").to(device)
            # exponential tail; the uniform is kept off 0 so no position gets p = 0 (ln 0 = -inf)
            e = -torch.log1p(-torch.rand(n, generator=gen, device="cpu").clamp_min(2.0 ** -24)).to(device)
            p = torch.where(spike, 0.5 + u, e)
            ss, ts = p[spike].sum(), p[~spike].sum()
            p = torch.where(spike, p * (top_mass / ss), p * ((1 - top_mass) / ts))
        else:
            lg = temp * torch.randn(n, generator=gen, device="cpu").to(device)
            p = torch.softmax(lg, 0)
        rows[gi] = p
    return rows


def planted_layer(P: int, H: int, G: int, n_o: int, m: int, d: int, seed: int = 7, dtype=torch.bfloat16,
                  device="cpu", values="gaussian"):
    """Returns q [P,H,m,d], k [P,G,n_o+m,d], v [P,G,n_o+m,d] in `dtype` on `device`.

    values="gaussian": V ~ N(0, 1).  values="embedding": V = X W_v as the reference generator
    forms it (trace.hpp:203-261): X's rows carry every group's key block (the planted log-weight
    direction c_g,j u_g + 0.05 eps; window rows 0.1 eps) and every head's query block (window
    rows only), W_v,g ~ N(0, 1/D), D = (G + H) d -- so a position's value is correlated with the
    planted weights, as in the reference's traces.  (Small shapes only: X is [n_o + m, D].)"""
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed)
    dgen = torch.Generator(device=device)
    dgen.manual_seed(seed + 1)
    g = H // G
    q = torch.empty((P, H, m, d), dtype=dtype, device=device)
    k = torch.empty((P, G, n_o + m, d), dtype=dtype, device=device)
    v = torch.randn((P, G, n_o + m, d), generator=dgen, device=device, dtype=torch.float32).to(dtype)
    for p in range(P):
        rows = planted_rows(G, n_o, gen, device=device)
        u = torch.randn((G, d), generator=gen).to(device)
        u = u / u.norm(dim=1, keepdim=True)
        c = torch.log(rows) + math.log(n_o)                                   # [G, n_o]
        kk = c[:, :, None] * u[:, None, :] + 0.05 * torch.randn((G, n_o, d), generator=dgen, device=device)
        kw = 0.1 * torch.randn((G, m, d), generator=dgen, device=device)
        k[p] = torch.cat([kk, kw], dim=1).to(dtype)
        uq = u.repeat_interleave(g, dim=0)                                     # [H, d]
        qq = math.sqrt(d) * uq[:, None, :] + 0.15 * torch.randn((H, m, d), generator=dgen, device=device)
        q[p] = qq.to(dtype)
        if values == "embedding":
            D = (G + H) * d
            x = torch.zeros((n_o + m, G + H, d), device=device)
            x[:, :G] = torch.cat([kk, kw], dim=1).transpose(0, 1)             # key blocks
            x[n_o:, G:] = qq.transpose(0, 1)                                  # query blocks (window rows)
            wv = torch.randn((G, D, d), generator=dgen, device=device) / math.sqrt(D)
            v[p] = torch.einsum("nD,gDe->gne", x.reshape(n_o + m, D), wv).to(dtype)
    return q, k, v
