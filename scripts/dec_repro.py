import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_11550_b200 as A
from paper_2407_11550_b200.synthetic import planted_layer
dev = torch.device("cuda:0")
P = int(os.environ.get("P", "8")); n = int(os.environ.get("N", "16384")); bud = int(os.environ.get("BUD", "4096"))
q, k, v = planted_layer(P, 32, 8, n - 32, 32, 128, seed=3, dtype=torch.bfloat16, device=dev)
cache = A.compress(q, k, v, bud * 8, reserve=2)
torch.cuda.synchronize()
print("cluster", A.lib().adakv_debug_decode_cluster(P, 8), "max seg", int(cache.seqlens.max()))
qd = torch.randn((P, 32, 128), device=dev).to(torch.bfloat16)
o = A.decode(qd, cache)
torch.cuda.synchronize()
print("ok", float(o.float().abs().mean()))
bad = torch.isnan(o.float()).any(dim=-1)
print("nan (p, h):", bad.nonzero().tolist()[:20])
print("seqlens:", cache.seqlens.view(P, 8).tolist())
kr, vr = cache.segment(6, 4)
print("seg nan K/V:", bool(torch.isnan(kr.float()).any()), bool(torch.isnan(vr.float()).any()), "inf:", bool(torch.isinf(kr.float()).any()), bool(torch.isinf(vr.float()).any()))
s = (qd[6, 16:20].float() @ kr.float().T) / 128 ** 0.5
print("logit max", float(s.max()), "min", float(s.min()))
p_ = torch.softmax(s, dim=-1)
ref = p_ @ vr.float()
print("ref nan", bool(torch.isnan(ref).any()), "out", o[6, 16, :4].tolist(), "ref", ref[0, :4].tolist())
