"""Print the per-phase timing of one dp_plan launch (cluster 0) at the bench
shape: python tools/plan_timing.py [context] [G]"""
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
from tools.gpu_warm import clocks, warm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if len(sys.argv) > 3:
    N.lib().dp_debug_set(1, int(sys.argv[3]))  # force the plan cluster size
k, v, c = generate_layer(1, 8, n, 128)
lay = cluster_layer(k, v)
q = torch.from_numpy(generate_queries(c, G, 1)[0]).cuda().to(torch.bfloat16)
ws = DecodeWorkspace(lay, G)
if os.environ.get('PLAN_DBG'):
    N.lib().dp_debug_set(10, int(os.environ['PLAN_DBG']))  # knob builds: A/B switches
lib = N.lib()
view = lay.view()
warm()
print('clocks after warm-up:', clocks())
for it in range(3):
    N.check(lib.dp_plan(view, N.ptr(q), 1, G, 1 / math.sqrt(128), 0.95, 0.7, N.ptr(ws.log_mass), None,
                        N.ptr(ws.counts), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(),
                        torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 384)()
lib.dp_debug_plan_timing(ctypes.cast(buf, ctypes.c_void_p))
t = np.array(buf[:], dtype=np.float64).reshape(16, 24)[:, [0, 1, 2, 14, 22, 13, 11, 21, 12, 23, 10, 3, 4, 20, 5, 6, 15, 7, 8, 16, 17, 18, 19, 9]]
nr = 16 if t[8:, 0].min() > 0 else 8
t = t[:nr]
t0 = t[:, 0].min()
names = ["start", "loads", "S", "t0in", "rb0", "mma0", "t0done", "t1in", "t1done", "t3in", "score", "P1", "A", "selin", "P2", "B", "cnts", "P3", "C", "offs", "lmst", "scan4", "rows", "P4"]
print("ncand (stats unavailable); see counts")
print("rank " + " ".join(f"{x:>6s}" for x in names))
for r in range(nr):
    print(f"{r:4d} " + " ".join(f"{(x - t0) / 1e3:6.2f}" if x > 0 else "     -" for x in t[r]))
cbuf = (ctypes.c_ulonglong * 32)()
lib.dp_debug_plan_clock(ctypes.cast(cbuf, ctypes.c_void_p))
cl = np.array(cbuf[:], dtype=np.float64).reshape(16, 2)
tt = np.array(buf[:], dtype=np.float64).reshape(16, 24)
print("SM clock inside the kernel (MHz):", [float((cl[r, 1] - cl[r, 0]) / (tt[r, 9] - tt[r, 0]) * 1e3) for r in range(nr)])
print("counts", ws.counts[0, :G].tolist(), "stats", ws.stats[0, 0].tolist())

