"""Host overhead per sparse_attention call (eager API) vs the raw C-ABI call."""
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer, sparse_attention  # noqa: E402
from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200.workload import generate_layer, generate_queries  # noqa: E402

k, v, c = generate_layer(1, 8, 4096, 128)
lay = cluster_layer(k, v)
q = torch.from_numpy(generate_queries(c, 4, 1)[0]).cuda().to(torch.bfloat16)
ws = DecodeWorkspace(lay, 4)
out = torch.empty_like(ws.out)
for _ in range(20):
    sparse_attention(q, lay, 0.95, 0.7, workspace=ws, out=out)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    sparse_attention(q, lay, 0.95, 0.7, workspace=ws, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"sparse_attention eager: {(t1 - t0) / n * 1e6:.2f} us per call (host issue)")
lib = N.lib()
view = lay.view()
args = (view, N.ptr(q), 1, 4, 1 / math.sqrt(128), 0.95, 0.7, N.ptr(ws.log_mass), N.ptr(ws.state), N.ptr(ws.counts),
        N.ptr(out), N.ptr(ws.lse), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(), torch.cuda.current_stream().cuda_stream)
t0 = time.perf_counter()
for _ in range(n):
    lib.dp_decode_step(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"raw dp_decode_step: {(t1 - t0) / n * 1e6:.2f} us per call (host issue)")
t0 = time.perf_counter()
for _ in range(n):
    torch.cuda.current_stream().cuda_stream
t1 = time.perf_counter()
print(f"current_stream lookup: {(t1 - t0) / n * 1e6:.2f} us")
