"""AKVC v1 export / import of compressed device caches.

The reference persists a FlattenedCache as (flat_cache.hpp:131-178, serde.hpp):
    "AKVC", u32 version = 1, u32 h, u32 d_h, u64 lengths[h],
    then data as little-endian f64: per head all key rows, then all value rows.
The device cache stores one segment per (problem, KV group) in separate K and V planes
(DESIGN.md §3).  `export_akvc` writes one problem (layer) in the reference layout -- either
one head per KV group or, like the reference's evict_layer result, one head per query head
(each member head repeats its group's rows, policies.hpp:276) -- so parity artefacts are
byte-comparable with files the reference writes.  `import_akvc` reads such a file back into a
device cache (one segment per head) that `ops.decode` can run on.
"""
from __future__ import annotations

import struct

import numpy as np
import torch

from . import _lib as L

MAGIC = b"AKVC"
VERSION = 1


def _flatten_bytes(heads_k, heads_v, d: int) -> bytes:
    lengths = [int(k.shape[0]) for k in heads_k]
    out = [MAGIC, struct.pack("<III", VERSION, len(lengths), d), struct.pack(f"<{len(lengths)}Q", *lengths)]
    for k, v in zip(heads_k, heads_v):
        out.append(np.ascontiguousarray(k.detach().to(torch.float64).cpu().numpy(), dtype="<f8").tobytes())
        out.append(np.ascontiguousarray(v.detach().to(torch.float64).cpu().numpy(), dtype="<f8").tobytes())
    return b"".join(out)


def export_akvc(cache, p: int = 0, per_query_head: bool = True) -> bytes:
    """Bytes of problem p of `cache` (ops.CompressedCache) in the AKVC v1 format.

    per_query_head=True: H heads, head i holding group i // (H/G)'s rows (the reference's
    evict_layer retained cache); False: G heads, one per KV group."""
    if not 0 <= p < cache.P:
        raise L.OutOfRange(2, "export_akvc: problem index out of range")
    segs = [cache.segment(p, g) for g in range(cache.G)]
    if per_query_head:
        gs = cache.H // cache.G
        segs = [segs[i // gs] for i in range(cache.H)]
    return _flatten_bytes([s[0] for s in segs], [s[1] for s in segs], cache.d)


def save_akvc(cache, path: str, p: int = 0, per_query_head: bool = True) -> None:
    data = export_akvc(cache, p, per_query_head)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:  # IoError (serde.hpp:24-27)
        raise L.IoError(4, f"cannot open for writing: {path} ({e})") from e


def parse_akvc(data: bytes):
    """(d_h, [lengths], K rows per head, V rows per head) as float64 numpy arrays; raises the
    FormatError equivalent on malformed input (flat_cache.hpp:153-168)."""
    if len(data) < 4:
        raise L.FormatError(3, "load_flattened: truncated header")
    if data[:4] != MAGIC:
        raise L.FormatError(3, "load_flattened: bad magic")
    if len(data) < 16:
        raise L.FormatError(3, "unexpected end of file")
    version, h, d = struct.unpack_from("<III", data, 4)
    if version != VERSION:
        raise L.FormatError(3, f"load_flattened: unsupported version {version}")
    pos = 16
    if len(data) < pos + 8 * h:
        raise L.FormatError(3, "unexpected end of file")
    lengths = list(struct.unpack_from(f"<{h}Q", data, pos))
    pos += 8 * h
    total = 2 * sum(lengths) * d
    if len(data) < pos + 8 * total:
        raise L.FormatError(3, "unexpected end of file")
    flat = np.frombuffer(data, dtype="<f8", count=total, offset=pos)
    ks, vs, o = [], [], 0
    for ln in lengths:
        ks.append(flat[o:o + ln * d].reshape(ln, d))
        o += ln * d
        vs.append(flat[o:o + ln * d].reshape(ln, d))
        o += ln * d
    return d, lengths, ks, vs


def import_akvc(data: bytes, device, dtype=torch.bfloat16, reserve: int = 0):
    """A device cache (ops.CompressedCache, P = 1, one segment per stored head, g = 1) holding
    the file's rows, with `reserve` spare rows per segment for decode appends."""
    from .ops import CompressedCache
    d, lengths, ks, vs = parse_akvc(data)
    h = len(lengths)
    caps = [ln + reserve for ln in lengths]
    rows = max(sum(caps), 1)
    kp = torch.zeros((rows, d), dtype=dtype, device=device)
    vp = torch.zeros((rows, d), dtype=dtype, device=device)
    starts = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int32) if h else np.zeros(0, np.int32)
    for i in range(h):
        s = int(starts[i])
        kp[s:s + lengths[i]] = torch.from_numpy(ks[i].copy()).to(device=device, dtype=dtype)
        vp[s:s + lengths[i]] = torch.from_numpy(vs[i].copy()).to(device=device, dtype=dtype)
    return CompressedCache(k=kp, v=vp, seg_start=torch.as_tensor(starts, device=device),
                           seqlens=torch.as_tensor(np.asarray(lengths, np.int32), device=device),
                           budgets=torch.as_tensor(np.asarray(lengths, np.int32), device=device),
                           P=1, H=h, G=h, m=0, d=d, reserve=reserve, layer_budget=int(sum(lengths)))
