"""How long the first flashinfer trtllm-gen / xqa decode call takes in a fresh process (kernel loading)."""
import time
t0 = time.time()
import torch
import flashinfer
from flashinfer.decode import trtllm_batch_decode_with_kv_cache
print("import", round(time.time() - t0, 1), flashinfer.__version__, flush=True)
n, H, G, d, P = 32768, 8, 4, 128, 64
k = torch.randn(H, n, d, device="cuda", dtype=torch.bfloat16)
v = torch.randn(H, n, d, device="cuda", dtype=torch.bfloat16)
q = torch.randn(1, H * G, d, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
bt = torch.arange(n // P, dtype=torch.int32, device="cuda").unsqueeze(0)
sl = torch.tensor([n], dtype=torch.int32, device="cuda")
pages = lambda t: torch.as_strided(t, (n // P, H, P, d), (P * d, n * d, d, 1))  # noqa: E731
for i in range(3):
    t0 = time.time()
    o = trtllm_batch_decode_with_kv_cache(q, (pages(k), pages(v)), ws, bt, sl, n, bmm1_scale=d ** -0.5)
    torch.cuda.synchronize()
    print("trtllm call", i, round(time.time() - t0, 2), "s", flush=True)
try:
    from flashinfer.decode import xqa_batch_decode_with_kv_cache
    for i in range(2):
        t0 = time.time()
        o2 = xqa_batch_decode_with_kv_cache(q, (pages(k), pages(v)), ws, bt, sl, n, bmm1_scale=d ** -0.5)
        torch.cuda.synchronize()
        print("xqa call", i, round(time.time() - t0, 2), "s", (o2.float() - o.float()).abs().max().item(), flush=True)
except Exception as e:
    print("xqa failed", repr(e)[:300])
