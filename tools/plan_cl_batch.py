"""Plan kernel time (in a CUDA graph) at batch > 1 for forced cluster sizes.

    python tools/plan_cl_batch.py [batch] [context]
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
H, G, d = 8, 4, 128
k, v, c = generate_layer(B, H, n, d)
lay = cluster_layer(k, v)
del k, v
q = torch.from_numpy(generate_queries(c, G, 1)[0]).cuda().to(torch.bfloat16)
ws = DecodeWorkspace(lay, G)
lib = N.lib()
view = lay.view()


def plan():
    N.check(lib.dp_plan(view, N.ptr(q), 1, G, 1 / math.sqrt(d), 0.95, 0.7, N.ptr(ws.log_mass), None,
                        N.ptr(ws.counts), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(),
                        torch.cuda.current_stream().cuda_stream))


for cl in (0, 4, 5, 6, 8, 10):
    lib.dp_debug_set(1, cl)
    plan()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            plan()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"B={B} n={n} CL={cl or 'auto'} (picked {lib.dp_debug_plan_occupancy(view, G, 0)}): "
          f"{e0.elapsed_time(e1) * 1e3 / 50:.1f} us per plan")
lib.dp_debug_set(1, 0)
