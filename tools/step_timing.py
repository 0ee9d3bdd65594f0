"""Per-kernel in-graph timing of the decode step (profiling aid).

    python tools/step_timing.py [context] [layers] [G]
(The phase-skip switches exist only in a knob build:
    DP_EXTRA_FLAGS=-DDP_AB_KNOBS python -m paper_2602_05191_b200.build --force)

Builds `layers` synthetic layers, then times CUDA graphs of: the plan alone
(one layer repeated / layers cycled), the attention alone (cycled), the full
plan + attend step (cycled) and the dense kernel (cycled).  Prints us per
layer for each.
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16
G = int(sys.argv[3]) if len(sys.argv) > 3 else 4
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
if os.environ.get("DP_SHARED_WS"):  # one workspace reused by every layer (a serving engine's layout)
    wss = [wss[0]] * L
views = [lay.view() for lay in layers]
lib = N.lib()
if os.environ.get("DP_HINT_TAU") is not None:  # L2 warm-up threshold (nats); 0 disables
    lib.dp_debug_set(8, int(round(10 * float(os.environ["DP_HINT_TAU"]))))
if os.environ.get("DP_SEG_COST") is not None:  # attention range balancing: rows per head-segment start
    lib.dp_debug_set(9, int(os.environ["DP_SEG_COST"]))
sc = 1.0 / math.sqrt(d)


def plan(i, j=None):
    j = i if j is None else j
    ws = wss[j]
    N.check(lib.dp_plan(views[j], N.ptr(qs[j]), 1, G, sc, 0.95, 0.7, N.ptr(ws.log_mass), None, N.ptr(ws.counts),
                        N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), torch.cuda.current_stream().cuda_stream))


def attend(j):
    ws = wss[j]
    N.check(lib.dp_attend(views[j], N.ptr(qs[j]), 1, G, sc, N.ptr(ws.log_mass), N.ptr(ws.out), N.ptr(ws.lse),
                          N.ptr(ws.ws), ws.ws.numel(), torch.cuda.current_stream().cuda_stream))


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


for j in range(L):
    plan(j)
    attend(j)
torch.cuda.synchronize()
print("max active plan clusters by size:", {c: lib.dp_debug_plan_occupancy(views[0], G, c) for c in (8, 9, 10, 11, 12, 14, 16)},
      "picked:", lib.dp_debug_plan_occupancy(views[0], G, 0))
if len(sys.argv) > 4:
    lib.dp_debug_set(1, int(sys.argv[4]))
print(f"context {n}, layers {L}, G {G}: us per layer")
print(f"  plan (same layer)     {timed(lambda: [plan(0) for _ in range(L)]):8.2f}")
print(f"  plan (layers cycled)  {timed(lambda: [plan(j) for j in range(L)]):8.2f}")
print(f"  attend (cycled)       {timed(lambda: [attend(j) for j in range(L)]):8.2f}")
print(f"  attend (same layer)   {timed(lambda: [attend(0) for j in range(L)]):8.2f}   (rows L2-resident)")
print(f"  plan+attend (cycled)  {timed(lambda: [(plan(j), attend(j)) for j in range(L)]):8.2f}")
print(f"  dense (cycled)        {timed(lambda: [dense(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(0, 1)
print(f"  attend stream-only    {timed(lambda: [attend(j) for j in range(L)]):8.2f}")
print(f"  dense stream-only     {timed(lambda: [dense(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(0, 0)
st = wss[0].stats[0].cpu().tolist()
print("  stats (rows, approx, chunks, exact clusters) of layer 0:", st)

# attention phase stamps of the last launch in the full-step graph (layer L-1)
import ctypes  # noqa: E402
import numpy as np  # noqa: E402

timed(lambda: [(plan(j), attend(j)) for j in range(L)], reps=1)
abuf = (ctypes.c_ulonglong * (512 * 12))()
lib.dp_debug_attn_timing(ctypes.cast(abuf, ctypes.c_void_p))
a = np.array(abuf[:], dtype=np.float64).reshape(512, 12)[:148]
rows = a[:, 7].copy(); segs = a[:, 8].copy(); pe = a[:, 9].copy(); pi = a[:, 10].copy(); a = a[:, :7]
a0 = a[:, 0].min()
rel = (a - a0) / 1e3
print("attn phases of the last step (us, rel. to first CTA start): start, prefix, first data, loop done, flushed, exit")
for name, col in (("start", 0), ("prefix", 1), ("data0", 2), ("loop", 3), ("flush", 4), ("merge0", 6),
                  ("exit", 5)):
    x = rel[:, col]
    x = x[(x > -1e6) & (x < 1e6)]
    if x.size:
        print(f"  {name:7s} min {x.min():7.2f} med {np.median(x):7.2f} max {x.max():7.2f}  (n={x.size})")
pbuf = (ctypes.c_ulonglong * 384)()
lib.dp_debug_plan_timing(ctypes.cast(pbuf, ctypes.c_void_p))
pt = np.array(pbuf[:], dtype=np.float64).reshape(16, 24)
pend = pt[:, 9][pt[:, 9] > 0]
pstart = pt[:, 0][pt[:, 0] > 0]
if pend.size:
    print(f"  plan cluster 0 (same layer): start {(pstart.min() - a0) / 1e3:.2f}, end max {(pend.max() - a0) / 1e3:.2f} us")
pe_rel = (pe - a0) / 1e3
pi_rel = (pi - a0) / 1e3
print(f"  producer: first row entries med {np.median(pe_rel):.2f}, first tile issued med {np.median(pi_rel):.2f}")
loop_end = rel[:, 3] - rel[:, 2]
for sg in (1, 2):
    sel = segs == sg
    if sel.any():
        print(f"  CTAs with {sg} head segment(s): n={int(sel.sum())} rows med {np.median(rows[sel]):.0f} "
              f"loop(data0->done) med {np.median(loop_end[sel]):.2f} max {loop_end[sel].max():.2f} us")
if os.environ.get("ATTN_PER_CTA"):  # every CTA: id, segments, rows, data0, loop done (cumulative rows -> head)
    cum = np.cumsum(rows)
    for c in range(rows.size):
        print(f"    cta {c:3d} seg {int(segs[c])} rows {int(rows[c]):5d} cum {int(cum[c]):7d} data0 {rel[c, 2]:7.2f} done {rel[c, 3]:7.2f} loop {rel[c, 3] - rel[c, 2]:6.2f}")
slow = np.argsort(-rel[:, 3])[:6]
print("  slowest CTAs (id, segments, rows, data0, loop done):",
      [(int(c), int(segs[c]), int(rows[c]), round(rel[c, 2], 2), round(rel[c, 3], 2)) for c in slow])
mer = np.where((rel[:, 6] > 0) & (rel[:, 6] < 1e3))[0]
for c in mer:
    print(f"  merging CTA {c}: loop {rel[c,3]:.2f} flush {rel[c,4]:.2f} "
          f"merge0 {rel[c,6]:.2f} exit {rel[c,5]:.2f}")
