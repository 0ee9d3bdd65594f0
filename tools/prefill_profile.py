"""Kernel-time breakdown of the prefill clustering of one layer (torch profiler).

    python tools/prefill_profile.py [context] [heads] [tc]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05191_b200 import cluster_layer  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H = int(sys.argv[2]) if len(sys.argv) > 2 else 8
tc = len(sys.argv) > 3 and sys.argv[3] == "tc"
if os.environ.get("DP_PP_SINGLE"):
    from paper_2602_05191_b200 import _native as N
    N.lib().dp_debug_set(3, 1)
k, v, _ = generate_layer(1, H, n, 128)
cluster_layer(k, v, max_iters=2, fp64_assign=False, tensor_cores=tc)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    cluster_layer(k, v, fp64_assign=False, tensor_cores=tc)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14))
