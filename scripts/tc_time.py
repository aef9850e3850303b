"""Times window scoring alone (graph replay) at the config-2 layer shape."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2407_11550_b200 as A
from paper_2407_11550_b200.synthetic import planted_layer
from kbench import graph_time
L = A.lib(); dev = torch.device("cuda:0")
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1
q, k, v = planted_layer(P, 32, 8, 32736, 32, 128, seed=11, dtype=torch.bfloat16, device=dev)
gs = torch.empty((P, 8, 32736), dtype=torch.float32, device=dev)
shape = A.ops.layer_shape(P, 32, 8, 32, 32736, 128)
nb = C.c_size_t(); A._lib.check(L.adakv_window_scores_workspace(2, C.byref(shape), C.byref(nb)))
ws = torch.zeros(nb.value * 2, dtype=torch.uint8, device=dev)
def k1():
    A._lib.check(L.adakv_window_scores(2, C.byref(shape), 7, 1, C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), None,
        C.c_void_p(gs.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
t = graph_time(k1)
print(f"debug={os.environ.get('ADAKV_TC_DEBUG','0')} P={P}: {t/P*1e3:.1f} us/layer", flush=True)
