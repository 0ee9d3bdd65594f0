"""Time dense / sparse attention of one 32K layer (events, no profiler),
with and without the math (dp_debug_set(0, 1)): separates streaming from
compute.  python tools/attn_probe.py
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
from tools.gpu_warm import clocks, warm  # noqa: E402

L = 6
lays, qs = [], []
for li in range(L):
    k, v, c = generate_layer(1, 8, 32768, 128, layer=li)
    lays.append(cluster_layer(k, v, layer=li))
    qs.append(torch.from_numpy(generate_queries(c, 4, 1, layer=li)[0]).cuda().to(torch.bfloat16))
    del k, v
wss = [DecodeWorkspace(l, 4) for l in lays]
lib = N.lib()
st = torch.cuda.current_stream().cuda_stream
sc = 1 / math.sqrt(128)


def run(mode):
    for li in range(L):
        v, ws, q = lays[li].view(), wss[li], qs[li]
        if mode == "dense":
            N.check(lib.dp_dense_attention(v, N.ptr(q), 1, 4, sc, N.ptr(ws.out), N.ptr(ws.lse), N.ptr(ws.ws),
                                           ws.ws.numel(), st))
        else:
            N.check(lib.dp_plan(v, N.ptr(q), 1, 4, sc, 0.95, 0.7, N.ptr(ws.log_mass), None, N.ptr(ws.counts),
                                N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), st))
            if mode == "sparse":
                N.check(lib.dp_attend(v, N.ptr(q), 1, 4, sc, N.ptr(ws.log_mass), N.ptr(ws.out), N.ptr(ws.lse),
                                      N.ptr(ws.ws), ws.ws.numel(), st))


warm()
print('clocks after warm-up:', clocks())
for dbg in (0, 1):
    lib.dp_debug_set(0, dbg)
    for mode in ("dense", "plan", "sparse"):
        for _ in range(3):
            run(mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run(mode)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 / L * 1e3
        print(f"dbg={dbg} {mode:6s} {us:8.2f} us/layer")
lib.dp_debug_set(0, 0)
