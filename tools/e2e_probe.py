"""e2e of the DecodeGraph serving form at the bench shape for several output
copy granularities:  python tools/e2e_probe.py [context] [layers]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeGraph, DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
G, H, d = 4, 8, 128
dev = torch.device("cuda")
ks = torch.empty((L, H, n, d), dtype=torch.bfloat16, device=dev)
vs = torch.empty_like(ks)
qs = []
for li in range(L):
    k, v, c = generate_layer(1, H, n, d, layer=li, device=dev)
    ks[li], vs[li] = k[0], v[0]
    qs.append(torch.from_numpy(generate_queries(c, G, 1, layer=li)[0]).to(dev).to(torch.bfloat16))
big = cluster_layer(ks, vs, fp64_assign=False)
del ks, vs
layers = big.split()
ws = DecodeWorkspace(layers[0], G)
qd = torch.stack(qs)  # [L, 1, Hq, d]
qh = qd.cpu().pin_memory()
oh = torch.empty(qd.shape, dtype=torch.float32).pin_memory()
for every in (1, 4, 8, 16, 32):
    g = DecodeGraph(layers, qd.clone(), 0.95, 0.7, workspace=ws, host_q=qh, host_out=oh, out_every=every)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"out_every {every:2d}: {e0.elapsed_time(e1) * 1e3 / 20:8.1f} us per step (device-timed replay incl. copies)")
gd = DecodeGraph(layers, qd.clone(), 0.95, 0.7, workspace=ws)
for _ in range(5):
    gd.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    gd.replay()
e1.record()
torch.cuda.synchronize()
print(f"no host copies:  {e0.elapsed_time(e1) * 1e3 / 20:8.1f} us per step")
