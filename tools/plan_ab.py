"""A/B timing of the plan kernel's parts (dp_debug_set(10, bits): 2 skips the
selection, 4 the work lists) in a CUDA graph of back-to-back plan launches:
    python tools/plan_ab.py [context] [G]
(The phase-skip switches exist only in a knob build:
    DP_EXTRA_FLAGS=-DDP_AB_KNOBS python -m paper_2602_05191_b200.build --force)"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
L = 8
k, v, c = generate_layer(1, 8, n, 128)
lay = cluster_layer(k, v, fp64_assign=False)
q = torch.from_numpy(generate_queries(c, G, 1)[0]).cuda().to(torch.bfloat16)
ws = DecodeWorkspace(lay, G)
lib = N.lib()
view = lay.view()
sc = 1 / math.sqrt(128)


def plan():
    N.check(lib.dp_plan(view, N.ptr(q), 1, G, sc, 0.95, 0.7, N.ptr(ws.log_mass), None, N.ptr(ws.counts),
                        N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), torch.cuda.current_stream().cuda_stream))


def attend():
    N.check(lib.dp_attend(view, N.ptr(q), 1, G, sc, N.ptr(ws.log_mass), N.ptr(ws.out), N.ptr(ws.lse),
                          N.ptr(ws.ws), ws.ws.numel(), torch.cuda.current_stream().cuda_stream))


def timed(body, reps=30):
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


plan()
attend()
torch.cuda.synchronize()
print(f"context {n} G {G}: plan cluster size {lib.dp_debug_plan_occupancy(view, G, 0)}; us per launch in graph")
for bits, name in ((0, "full plan"), (32, "no centroid L2 prefetch"), (8, "no row expansion"), (4, "no work lists"), (2, "no selection"),
                   (6, "no selection, no lists"), (128, "launch + wait + q load only"), (64, "launch + wait only")):
    lib.dp_debug_set(10, bits)
    print(f"  {name:28s} {timed(lambda: [plan() for _ in range(L)]):7.2f}")
lib.dp_debug_set(10, 0)
print(f"  {'plan + attend':28s} {timed(lambda: [(plan(), attend()) for _ in range(L)]):7.2f}")
for bits, name in ((64, "attend: no approx rows"), (32, "attend: P hi only"), (1, "attend: no math"), (4, "attend: no merge"), (8, "attend: no counters/merge"),
                   (2, "attend: no flush/merge"), (3, "attend: neither")):
    lib.dp_debug_set(0, bits)
    print(f"  plan + {name:28s} {timed(lambda: [(plan(), attend()) for _ in range(L)]):7.2f}")
lib.dp_debug_set(0, 0)
print(f"  {'attend alone':28s} {timed(lambda: [attend() for _ in range(L)]):7.2f}")
for cl in (8, 10):
    lib.dp_debug_set(1, cl)
    print(f"  CL {cl:2d}: plan {timed(lambda: [plan() for _ in range(L)]):7.2f}  plan + attend "
          f"{timed(lambda: [(plan(), attend()) for _ in range(L)]):7.2f}")
lib.dp_debug_set(1, 0)
