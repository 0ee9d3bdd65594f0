import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer, sparse_attention
from paper_2602_05191_b200.workload import generate_layer
k, v, _ = generate_layer(1, 2, 4096, 128)
lay = cluster_layer(k, v, fp64_assign=False)
ws = DecodeWorkspace(lay, 4)
q = torch.full((1, 8, 128), float(sys.argv[1]), dtype=torch.bfloat16, device="cuda")
sparse_attention(q, lay, 0.95, 0.7, workspace=ws)
torch.cuda.synchronize()
print("ok", ws.counts[0].tolist(), ws.stats[0].tolist())
