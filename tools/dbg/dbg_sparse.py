import sys, math, torch, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import doublep_oracle as O
from paper_2602_05191_b200 import cluster_layer, sparse_attention, DecodeWorkspace
from paper_2602_05191_b200 import _native as N
spec = O.WorkloadSpec(context_len=2048, head_dim=128, num_kv_heads=2, gqa_group=4, num_steps=1, tail_profile='peaked', seed=0)
keys, values, queries = O.generate(spec)
k = torch.from_numpy(keys[0]).cuda().to(torch.bfloat16).unsqueeze(0)
v = torch.from_numpy(values[0]).cuda().to(torch.bfloat16).unsqueeze(0)
lay = cluster_layer(k, v)
q = torch.from_numpy(queries[0, 0]).cuda().to(torch.bfloat16).unsqueeze(0)
out, ws = sparse_attention(q, lay, 0.95, 0.7, return_plan=True)
torch.cuda.synchronize()
print("out norms", out[0].norm(dim=-1).tolist())
print("lse", ws.lse[0].tolist())
print("counts", ws.counts[0].tolist(), "stats", ws.stats[0].tolist())
wl_bytes = ws.ws
# decode workspace layout: runs, approx, cnt(4*BH ints), rowidx, counters, prefix, done, apart, partials
print("ws size", ws.ws.numel())
import ctypes
abuf = (ctypes.c_ulonglong * (512 * 8))()
N.lib().dp_debug_attn_timing(ctypes.cast(abuf, ctypes.c_void_p))
a = np.array(abuf[:], dtype=np.float64).reshape(512, 8)[:40]
t0 = a[a[:, 0] > 0, 0].min()
for i in range(34):
    print(i, ["%.2f" % ((x - t0) / 1e3) if x > 0 else "-" for x in a[i, :6]])
# workspace layout (decode_ws_layout): runs, approx, cnt, rowidx, counters, prefix, done, apart, partials
BH, cap, rc, G, d = 2, lay.cluster_cap, lay.row_cap, 4, 128
al = lambda x: (x + 255) & ~255
o = 0
o += al(BH * (cap + 2) * 16); o += al(BH * cap * 8); cnt_off = o; o += al(BH * 4 * 4)
row_off = o; o += al(BH * rc * 4); ctr_off = o; o += al(BH * 4)
wsb = ws.ws.cpu().numpy()
print("cnt", wsb[cnt_off:cnt_off + BH * 16].view(np.int32))
print("counters", wsb[ctr_off:ctr_off + BH * 4].view(np.int32))
print("rowidx head0[:8]", [hex(x) for x in wsb[row_off:row_off + 32].view(np.uint32)])
