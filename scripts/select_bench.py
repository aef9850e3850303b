"""Select-kernel latency over the score distributions SURVEY §8(d) asks for (radix pass count
depends on them): realistic planted-head scores, all-equal (maximum tie), quantised {k/64}
and underflowing tails (fp32 zeros).  Config-2 shape: G = 8 groups x 32736 positions, outside
budget 16128, adaptive + safeguard + repair, for P = 1 and P = 32 problems per launch.
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402
from scripts.kbench import graph_time  # noqa: E402

dev = torch.device("cuda:0")
G, n_o, m, H, d = 8, 32736, 32, 32, 128
total = 2048 * G - m * G
off = np.arange(G + 1, dtype=np.int64) * n_o
q, k, v = planted_layer(1, H, G, n_o, m, d, seed=11, dtype=torch.bfloat16, device=dev)
real = A.window_scores(q, k, 7).reshape(1, G * n_o).float()
gen = torch.Generator(device=dev)
gen.manual_seed(3)
dists = {
    "realistic": real,
    "all_equal": torch.full_like(real, 0.125),
    "quantised_k64": torch.floor(torch.rand(real.shape, generator=gen, device=dev) * 64) / 64,
    "underflow_tail": torch.where(torch.rand(real.shape, generator=gen, device=dev) < 0.9, torch.zeros_like(real), real),
}
res = {}
for name, s1 in dists.items():
    for P in (1, 32):
        s = s1.repeat(P, 1).contiguous()
        t = graph_time(lambda: A.segmented_select(s, off, total, "adaptive", blend=True, alpha=0.2, repair=True,
                                                  want_keep=False, want_pos=True), iters=10)
        res[f"{name}_P{P}_us"] = round(t * 1e3, 2)
print(json.dumps({"select_latency": res, "shape": {"G": G, "n_o": n_o, "outside_budget": total}}))
