"""Per-phase SM-cycle breakdown of one dp_plan launch (DP_PROFILE build):
    DP_PROFILE=1 python tools/plan_cycles.py [context] [G]
Prints, for every CTA of cluster 0, the cycles between consecutive phase
stamps (plan.cu stamp() events) and the select.cuh phases of the owners."""
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
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
k, v, c = generate_layer(1, 8, n, 128)
lay = cluster_layer(k, v)
q = torch.from_numpy(generate_queries(c, G, 1)[0]).cuda().to(torch.bfloat16)
ws = DecodeWorkspace(lay, G)
lib = N.lib()
for it in range(5):
    N.check(lib.dp_plan(lay.view(), N.ptr(q), 1, G, 1 / math.sqrt(128), 0.95, 0.7, N.ptr(ws.log_mass), None,
                        N.ptr(ws.counts), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(),
                        torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 384)()
lib.dp_debug_plan_cycles(ctypes.cast(buf, ctypes.c_void_p))
t = np.array(buf[:], dtype=np.float64).reshape(16, 24)
order = [0, 1, 2, 10, 3, 4, 20, 5, 6, 15, 7, 8, 16, 17, 18, 19, 9]
names = ["start", "loads", "S", "score", "P1", "A", "M", "P2", "B", "cnts", "P3", "C", "offs", "lmst", "scan4", "rows", "P4"]
CL = lib.dp_debug_plan_occupancy(lay.view(), G, 0)
print(f"context {n} G {G}: cluster size {CL}; us between consecutive stamps (1.965 GHz), per CTA of cluster 0")
print("rank " + " ".join(f"{x:>6s}" for x in names[1:]) + "   total")
for r in range(min(CL, 16)):
    row = t[r, order]
    prev, out = row[0], []
    for x in row[1:]:
        if x > 0:
            out.append(f"{(x - prev) / 1965:6.2f}")
            prev = x
        else:
            out.append("     -")
    print(f"{r:4d} " + " ".join(out) + f"  {(prev - row[0]) / 1965:6.2f}")
sb = (ctypes.c_ulonglong * 128)()
lib.dp_debug_sel_cycles(ctypes.cast(sb, ctypes.c_void_p))
s = np.array(sb[:], dtype=np.float64).reshape(16, 8)
sn = ["hist", "scan", "cand", "rank", "cut2", "states"]
print("select phases of the owner CTAs (us): " + " ".join(f"{x:>6s}" for x in sn))
for r in range(G):
    d = np.diff(s[r][:7]) / 1965
    print(f"{r:4d} " + " ".join(f"{x:6.2f}" for x in d))
if os.environ.get("DP_EXTRA_FLAGS", "").find("DP_SEL_REPEAT") >= 0:
    lib.dp_debug_sel_cycles2(ctypes.cast(sb, ctypes.c_void_p))
    s = np.array(sb[:], dtype=np.float64).reshape(16, 8)
    print("first (cold) pass of the repeated selection (us):")
    for r in range(G):
        d = np.diff(s[r][:7]) / 1965
        print(f"{r:4d} " + " ".join(f"{x:6.2f}" for x in d) + f"  total {(s[r,7]-s[r,0])/1965:6.2f}")
sb2 = (ctypes.c_ulonglong * 128)()
lib.dp_debug_sel_sub(ctypes.cast(sb2, ctypes.c_void_p))
s2 = np.array(sb2[:], dtype=np.float64).reshape(16, 8)
print("select phase-2 sub-steps (us from the phase start): loads, warp scan, sync1, warp0 scan+sync2, bins")
for r in range(G):
    print(f"{r:4d} " + " ".join(f"{(x - s[r][1]) / 1965:6.2f}" for x in s2[r][:5]))
