"""p sweep on one geometry (70B shape, 64 q / 8 kv heads,
128K): in-graph us per layer of the sparse step at each (p1, p2), the dense
kernel, and the union fraction.  python tools/psweep.py [context] [layers] [G]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
G = int(sys.argv[3]) if len(sys.argv) > 3 else 8
H, d = 8, 128
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
wss = [DecodeWorkspace(lay, G) for lay in layers]
views = [lay.view() for lay in layers]
lib = N.lib()
sc = 1.0 / math.sqrt(d)


def step(j, p1, p2):
    ws = wss[j]
    cs = torch.cuda.current_stream().cuda_stream
    N.check(lib.dp_plan(views[j], N.ptr(qs[j]), 1, G, sc, p1, p2, N.ptr(ws.log_mass), None, N.ptr(ws.counts),
                        N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), cs))
    N.check(lib.dp_attend(views[j], N.ptr(qs[j]), 1, G, sc, N.ptr(ws.log_mass), N.ptr(ws.out), N.ptr(ws.lse),
                          N.ptr(ws.ws), ws.ws.numel(), cs))


def dense(j):
    ws = wss[j]
    N.check(lib.dp_dense_attention(views[j], N.ptr(qs[j]), 1, G, sc, N.ptr(ws.out), N.ptr(ws.lse), N.ptr(ws.ws),
                                   ws.ws.numel(), torch.cuda.current_stream().cuda_stream))


def timed(body, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps / L


td = timed(lambda: [dense(j) for j in range(L)])
print(f"context {n}, G {G}, {L} layers: dense {td:.2f} us/layer")
for p1, p2 in [(0.9, 0.7), (0.95, 0.7), (0.99, 0.7), (0.99, 0.8)]:
    ts = timed(lambda: [step(j, p1, p2) for j in range(L)])
    st = wss[0].stats[0].cpu().double()
    u = float(st[:, 0].mean() / n)
    print(f"  p=({p1},{p2}): sparse {ts:.2f} us/layer  speedup {td / ts:.2f}x  union rows {u:.3f} of N")
