"""How well does a score threshold right after scoring (lm >= max - tau)
predict the exact (stage-2) clusters?  For each tau: fraction of the true
GQA-union exact rows covered and prefetched rows / true union rows.

    python tools/prefetch_tau.py [context] [layers] [profile]
"""
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
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prof = sys.argv[3] if len(sys.argv) > 3 else "peaked"
H, G, d = 8, 4, 128
lib = N.lib()
taus = [2, 3, 4, 5, 6, 8, 10, 12]
cov = {t: [] for t in taus}
ratio = {t: [] for t in taus}
for li in range(L):
    k, v, c = generate_layer(1, H, n, d, layer=li)
    lay = cluster_layer(k, v, fp64_assign=False)
    ws = DecodeWorkspace(lay, G)
    qs = generate_queries(c, G, 4, profile=prof, layer=li)
    offs = lay.offs[0].cpu().numpy().astype(np.int64)
    ncl = lay.nclusters[0].cpu().numpy()
    for s in range(4):
        q = torch.from_numpy(qs[s]).cuda().to(torch.bfloat16)
        st = torch.zeros_like(ws.state)
        N.check(lib.dp_plan(lay.view(), N.ptr(q), 1, G, 1 / math.sqrt(d), 0.95, 0.7, N.ptr(ws.log_mass), N.ptr(st),
                            N.ptr(ws.counts), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(),
                            torch.cuda.current_stream().cuda_stream))
        lm = ws.log_mass[0].cpu().numpy()
        stn = st[0].cpu().numpy()
        for h in range(H):
            K = int(ncl[h])
            sizes = np.diff(offs[h, :K + 1])
            lmh = lm[h * G:(h + 1) * G, :K]
            exact = (stn[h * G:(h + 1) * G, :K] == 2).any(0)
            gap = (lmh - lmh.max(1, keepdims=True)).max(0)  # best head's gap to its max
            urows = sizes[exact].sum()
            for t in taus:
                pre = gap >= -t
                cov[t].append(sizes[exact & pre].sum() / max(urows, 1))
                ratio[t].append(sizes[pre].sum() / max(urows, 1))
print(f"context {n} profile {prof}: tau -> union rows covered (mean/min), prefetched rows / union rows (mean/max)")
for t in taus:
    print(f"  tau {t:2d}: covered {np.mean(cov[t]):.3f} / {np.min(cov[t]):.3f}   prefetch ratio {np.mean(ratio[t]):.2f} / "
          f"{np.max(ratio[t]):.2f}")
