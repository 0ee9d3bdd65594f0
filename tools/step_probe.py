"""One-launch decode step vs the two-launch (plan + attend) path: agreement and
in-graph timing (profiling aid).

    python tools/step_probe.py [context] [layers] [G] [taus comma-separated, 0.1 nat units]

Builds `layers` synthetic layers (bench law), checks that dp_decode_step's
one-launch step gives the same selection and (to fp32 rounding) the same
outputs as plan + attend, then times CUDA graphs of all layers (cycled)
for both paths and for the dense kernel.  With DP_PROFILE=1 builds, prints
the step kernel's phase stamps of cluster 0.
"""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16
G = int(sys.argv[3]) if len(sys.argv) > 3 else 4
taus = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [60]
B = int(os.environ.get("BATCH", "1"))
H, d = 8, 128
dev = torch.device("cuda")
ks = torch.empty((L * B, H, n, d), dtype=torch.bfloat16, device=dev)
vs = torch.empty_like(ks)
qs = []
for li in range(L):
    k, v, c = generate_layer(B, H, n, d, layer=li, device=dev)
    ks[li * B:(li + 1) * B], vs[li * B:(li + 1) * B] = k, v
    qs.append(torch.from_numpy(generate_queries(c, G, 1, layer=li)[0]).to(dev).to(torch.bfloat16))
big = cluster_layer(ks, vs, fp64_assign=False)
del ks, vs
if B == 1:
    layers = big.split()
else:
    from paper_2602_05191_b200 import ClusteredLayer

    layers = []
    for li in range(L):
        sl = lambda t: t[li * B:(li + 1) * B]  # noqa: E731
        lay = ClusteredLayer(sl(big.keys), sl(big.values), sl(big.offs), sl(big.nclusters), sl(big.centroids),
                             sl(big.value_means), sl(big.perm), big.n_tokens, big.sink, big.window)
        layers.append(lay)
wss = [DecodeWorkspace(lay, G) for lay in layers]
views = [lay.view() for lay in layers]
lib = N.lib()
sc = 1.0 / math.sqrt(d)
print("step cluster size:", lib.dp_debug_step_cluster_size(views[0], G))


def step(j, ws=None):
    ws = wss[j] if ws is None else ws
    N.check(lib.dp_decode_step(views[j], N.ptr(qs[j]), 1, G, sc, 0.95, 0.7, N.ptr(ws.log_mass), N.ptr(ws.state),
                               N.ptr(ws.counts), N.ptr(ws.out), N.ptr(ws.lse), N.ptr(ws.stats), N.ptr(ws.ws),
                               ws.ws.numel(), torch.cuda.current_stream().cuda_stream))


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


# ---- agreement: one-launch step vs plan + attend --------------------------
worst, mism = 0.0, 0
ref = [DecodeWorkspace(lay, G) for lay in layers[:4]]
lib.dp_debug_set(6, 0)  # the one-launch step is opt-in
for j in range(min(4, L)):
    lib.dp_debug_set(6, 1)
    step(j, ref[j])
    lib.dp_debug_set(6, 0)
    step(j)
    torch.cuda.synchronize()
    a, b = wss[j], ref[j]
    K = int(layers[j].nclusters.max())
    mism += int((a.state[..., :K] != b.state[..., :K]).sum()) + int((a.counts != b.counts).sum())
    err = ((a.out - b.out).norm(dim=-1) / b.out.norm(dim=-1)).max().item()
    worst = max(worst, err)
    assert torch.equal(a.stats[..., [0, 1, 3]], b.stats[..., [0, 1, 3]]), (a.stats, b.stats)
    assert torch.allclose(a.log_mass, b.log_mass, rtol=0, atol=0)
print(f"one-launch vs plan+attend: state/count mismatches {mism}, worst output rel diff {worst:.2e}")

print(f"context {n}, batch {B}, layers {L}, G {G}: us per layer (graph, layers cycled)")
for tau in taus:
    lib.dp_debug_set(4, tau)
    print(f"  one-launch step tau={tau / 10:4.1f}  {timed(lambda: [step(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(4, 0)
lib.dp_debug_set(7, 1)
print(f"  one-launch, no attention math   {timed(lambda: [step(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(7, 2)
print(f"  one-launch, no K/V loads        {timed(lambda: [step(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(7, 3)
print(f"  one-launch, neither             {timed(lambda: [step(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(7, 0)
lib.dp_debug_set(4, taus[-1])
lib.dp_debug_set(6, 1)
print(f"  plan + attend            {timed(lambda: [step(j) for j in range(L)]):8.2f}")
lib.dp_debug_set(6, 0)
print(f"  dense                    {timed(lambda: [dense(j) for j in range(L)]):8.2f}")
st = wss[0].stats.view(-1, 4)[:H].cpu().tolist()
print("  stats (rows, approx, chunks, exact clusters) of layer 0:", st)

buf = (ctypes.c_ulonglong * 384)()
timed(lambda: [step(j) for j in range(L)], reps=1)
lib.dp_debug_step_timing(ctypes.cast(buf, ctypes.c_void_p))
allt = np.array(buf[:], dtype=np.float64)
t = allt[:256].reshape(16, 16)
sel = allt[256:].reshape(16, 8)
if t[0, 0] > 0:
    work = t[:, 11:14].copy()
    cl = lib.dp_debug_step_cluster_size(views[0], G)
    t = t[:cl, :11]
    t0 = t[:, 0].min()
    names = ["start", "S", "P1", "A", "P2", "B", "lists", "loop", "push", "C", "end"]
    print("step phases of the last launch, cluster 0 (us from the first CTA start)")
    print("rank " + " ".join(f"{x:>6s}" for x in names))
    for r in range(cl):
        print(f"{r:4d} " + " ".join(f"{(x - t0) / 1e3:6.2f}" if x > 0 else "     -" for x in t[r])
              + f"   rows {int(work[r, 0])} runs {int(work[r, 1])} approx {int(work[r, 2])}")
    print("selection phases of the owner CTAs (us from the first CTA start): start, hist, scan, b1, cmpct, rank, cut1, end")
    for r in range(G):
        print(f"{r:4d} " + " ".join(f"{(x - t0) / 1e3:6.2f}" if x > 0 else "     -" for x in sel[r]))
