"""Per-kernel view of the unfused dp_sparse_attention (worklist + approx
partial + attention) next to dp_plan + dp_attend at one shape, for ncu:
    python tools/sparse_attn_probe.py [context]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
G = 4
k, v, c = generate_layer(1, 8, n, 128)
lay = cluster_layer(k, v, fp64_assign=False)
q = torch.from_numpy(generate_queries(c, G, 1)[0]).cuda().to(torch.bfloat16)
ws = DecodeWorkspace(lay, G)
lib = N.lib()
view = lay.view()
sc = 1 / math.sqrt(128)
s = torch.cuda.current_stream().cuda_stream
for it in range(3):
    N.check(lib.dp_plan(view, N.ptr(q), 1, G, sc, 0.95, 0.7, N.ptr(ws.log_mass), N.ptr(ws.state), N.ptr(ws.counts),
                        N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), s))
    N.check(lib.dp_attend(view, N.ptr(q), 1, G, sc, N.ptr(ws.log_mass), N.ptr(ws.out), N.ptr(ws.lse), N.ptr(ws.ws),
                          ws.ws.numel(), s))
    N.check(lib.dp_sparse_attention(view, N.ptr(q), 1, G, sc, N.ptr(ws.log_mass), N.ptr(ws.state), N.ptr(ws.out),
                                    N.ptr(ws.lse), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), s))
torch.cuda.synchronize()
print("ok")
