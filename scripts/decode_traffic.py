"""DRAM traffic of ONE decode launch at a known step, beside that launch's algorithmic bytes.

Builds the config-2 compressed cache (bench.py's inputs: 32 layers, 32K prompt, budget
2048/head), runs `--step` decode steps (appends) so the caches have the length they have in
the middle of the bench's 512 steps, then launches the decode of layer `--layer` once more,
chained after layer-1's decode as in the bench.  Run it under
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:decode_tc -s <launches before> -c 1
(scripts/gpu_ncu.sh traffic); without ncu it prints the algorithmic bytes of that launch.
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_11550_b200 as A  # noqa: E402
from paper_2407_11550_b200 import pipeline as PL  # noqa: E402
from paper_2407_11550_b200.synthetic import planted_layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--step", type=int, default=256)
    ap.add_argument("--layer", type=int, default=16)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    L, H, G, d, m, n = 32, 32, 8, 128, 32, 32768
    LB = 2048 * G
    q, k, v = planted_layer(L, H, G, n - m, m, d, seed=1000, dtype=torch.bfloat16, device=dev)
    cache = PL.compress_model(q.view(L, 1, H, m, d), k.view(L, 1, G, n, d), v.view(L, 1, G, n, d), LB,
                              reserve=args.step + 2)
    del q, k, v
    max_rows = int(cache.seg_cap.max())
    dg = PL.DecodeGraph(cache, L, 1, max_rows, use_graph=False)
    lib = A.lib()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for s in range(args.step):  # advance every layer's caches by `step` appended rows
        dg.q.normal_()
        dg.k_new.normal_()
        dg.v_new.normal_()
        dg.step()
    torch.cuda.synchronize()
    rows = int(cache.seqlens[args.layer * G:(args.layer + 1) * G].sum()) + G  # incl. this launch's append
    nbytes = 2 * 2 * d * rows + 2 * 2 * H * d + 2 * 2 * G * d
    # the measured launch: layer-1 then `layer`, chained as in the bench
    PL.decode_layer(lib, cache, args.layer - 1, 1, dg.q[args.layer - 1], dg.k_new[args.layer - 1],
                    dg.v_new[args.layer - 1], dg.out[args.layer - 1], dg.ws, max_rows, st, chained=False)
    PL.decode_layer(lib, cache, args.layer, 1, dg.q[args.layer], dg.k_new[args.layer], dg.v_new[args.layer],
                    dg.out[args.layer], dg.ws, max_rows, st, chained=True)
    torch.cuda.synchronize()
    print(json.dumps({"step": args.step, "layer": args.layer, "rows_attended": rows,
                      "algorithmic_bytes": nbytes, "launches_before": args.step * L + 1}))


if __name__ == "__main__":
    main()
