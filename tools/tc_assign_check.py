"""Tensor-core (tcgen05) k-means assignment vs the FFMA fp32 and DFMA fp64
paths on one bf16 layer: agreement of final assignments/objective and timing.

    python tools/tc_assign_check.py [context] [heads] [iters]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import cluster_layer  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H = int(sys.argv[2]) if len(sys.argv) > 2 else 8
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 25
k, v, _ = generate_layer(1, H, n, 128)
res = {}
for name, kw in (("fp64", dict(fp64_assign=True)), ("fp32", dict(fp64_assign=False)),
                 ("tc", dict(fp64_assign=False, tensor_cores=True))):
    cluster_layer(k, v, max_iters=1, **kw)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lay = cluster_layer(k, v, max_iters=iters, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    it = lay.iters.cpu()
    obj = lay.objective.cpu()
    last = torch.stack([obj[i, it[i] - 1] for i in range(obj.shape[0])])
    res[name] = (lay, last)
    print(f"{name:5s} {dt * 1e3:8.1f} ms  iters {it.tolist()}  final objective {last[:3].tolist()}")
for name in ("fp32", "tc"):
    a, b = res[name][0].perm.cpu(), res["fp64"][0].perm.cpu()
    same = (a == b).float().mean().item()
    rel = ((res[name][1] - res["fp64"][1]).abs() / res["fp64"][1]).max().item()
    print(f"{name} vs fp64: identical row order {same:.6f}, max objective rel diff {rel:.2e}")
# one iteration from identical seeding: assignment agreement
one = {}
for name, kw in (("fp64", dict(fp64_assign=True)), ("fp32", dict(fp64_assign=False)),
                 ("tc", dict(fp64_assign=False, tensor_cores=True))):
    lay = cluster_layer(k, v, max_iters=1, **kw)
    one[name] = (lay.offs.cpu(), lay.perm.cpu(), lay.objective.cpu()[:, 0])
for name in ("fp32", "tc"):
    same = (one[name][0] == one["fp64"][0]).all().item() and (one[name][1] == one["fp64"][1]).float().mean().item()
    rel = ((one[name][2] - one["fp64"][2]).abs() / one["fp64"][2]).max().item()
    print(f"1 iteration {name} vs fp64: same layout {same}, objective rel diff {rel:.2e}")
