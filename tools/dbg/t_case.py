import time, sys, torch, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from oracle import doublep_oracle as O
from paper_2602_05191_b200 import cluster_layer, sparse_attention
for (n, H, G, d, dt, B) in [(300, 2, 4, 128, torch.float32, 3), (1500, 3, 8, 128, torch.bfloat16, 1), (6000, 1, 8, 128, torch.float32, 2)]:
    ks=[];vs=[];qs=[]
    t0=time.time()
    for b in range(B):
        spec = O.WorkloadSpec(context_len=n, head_dim=d, num_kv_heads=H, gqa_group=G, num_steps=1, tail_profile='mixed', seed=5+b)
        k, v, q = O.generate(spec); ks.append(k[0]); vs.append(v[0]); qs.append(q[0,0])
    t1=time.time()
    kd=torch.from_numpy(np.stack(ks)).cuda().to(dt); vd=torch.from_numpy(np.stack(vs)).cuda().to(dt); q=torch.from_numpy(np.stack(qs)).cuda().to(dt)
    torch.cuda.synchronize(); t2=time.time()
    lay=cluster_layer(kd, vd, fp64_assign=False); torch.cuda.synchronize(); t3=time.time()
    out, ws = sparse_attention(q, lay, 0.9, 0.7, return_plan=True); torch.cuda.synchronize(); t4=time.time()
    print(n, H, G, d, dt, B, f"gen {t1-t0:.2f} upload {t2-t1:.2f} cluster {t3-t2:.2f} attn {t4-t3:.2f}", flush=True)
