import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from oracle import doublep_oracle as O
from paper_2602_05191_b200 import _native as N, cluster_layer, sparse_attention
for (n, H, G, cl) in [(300, 3, 6, 12), (300, 3, 6, 0), (300, 3, 6, 8), (300, 3, 4, 12), (300, 1, 6, 12), (700, 3, 6, 12), (300, 3, 8, 12), (300, 3, 6, 16)]:
    spec = O.WorkloadSpec(context_len=n, head_dim=128, num_kv_heads=H, gqa_group=G, num_steps=1, tail_profile="uniform", seed=1)
    k, v, q = O.generate(spec)
    kd = torch.from_numpy(k[0]).cuda().to(torch.bfloat16).unsqueeze(0); vd = torch.from_numpy(v[0]).cuda().to(torch.bfloat16).unsqueeze(0)
    qd = torch.from_numpy(q[0, 0]).cuda().to(torch.bfloat16).unsqueeze(0)
    N.lib().dp_debug_set(1, cl)
    lay = cluster_layer(kd, vd, fp64_assign=False)
    try:
        out = sparse_attention(qd, lay, 0.5, 0.3); torch.cuda.synchronize(); print(n, H, G, cl, "ok", lay.cluster_cap)
    except Exception as e:
        print(n, H, G, cl, "ERR", e, lay.cluster_cap)
