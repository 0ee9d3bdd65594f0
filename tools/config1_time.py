"""Config 1 on the GPU: one layer, 32 q / 8 kv heads, d = 128,
8K tokens, fp32 cache, reference generator law; in-graph us per decode step of
the product call (dp_decode_step) and of the dense kernel.
    python tools/config1_time.py [profile]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import doublep_oracle as O  # noqa: E402

from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer, dense_attention, sparse_attention  # noqa: E402

prof = sys.argv[1] if len(sys.argv) > 1 else "peaked"
spec = O.WorkloadSpec(context_len=8192, head_dim=128, num_kv_heads=8, gqa_group=4, num_steps=8, tail_profile=prof,
                      seed=0)
keys, values, queries = O.generate(spec)
k = torch.from_numpy(keys[0][None]).cuda()
v = torch.from_numpy(values[0][None]).cuda()
lay = cluster_layer(k, v)
qs = [torch.from_numpy(queries[s, 0][None]).cuda() for s in range(queries.shape[0])]
ws = DecodeWorkspace(lay, 4)


def timed(fn):
    for s in range(3):
        fn(qs[s])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn(qs[0])
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for s in range(8):
            fn(qs[s])
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / 20 / 8


sp = timed(lambda q: sparse_attention(q, lay, 0.95, 0.7, workspace=ws))
de = timed(lambda q: dense_attention(q, lay, workspace=ws))
print(f"config 1 ({prof}, fp32 cache, 8K, 32q/8kv, d128): sparse {sp:.1f} us/step, dense {de:.1f} us/step")
