"""Dense decode comparators from the installed FlashInfer (library code,
timed like our kernels: CUDA graph over 8 layers, us per layer):
single_decode_with_kv_cache and trtllm_batch_decode_with_kv_cache (the
trtllm-gen Blackwell kernels) on a strided page view of a [H, N, d] cache."""
import torch
import flashinfer
from flashinfer.decode import trtllm_batch_decode_with_kv_cache

print(flashinfer.__version__)


def timed(fn, L, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for j in range(L):
            fn(j)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(L):
            fn(j)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps / L


for n in (32768, 131072):
    H, G, d, L, P = 8, 4, 128, 6, 64
    ks = [torch.randn(H, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(L)]
    vs = [torch.randn(H, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(L)]
    q = torch.randn(1, H * G, d, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    bt = torch.arange(n // P, dtype=torch.int32, device="cuda").unsqueeze(0)
    sl = torch.tensor([n], dtype=torch.int32, device="cuda")
    pages = lambda t: torch.as_strided(t, (n // P, H, P, d), (P * d, n * d, d, 1))  # noqa: E731
    kp = [pages(k) for k in ks]
    vp = [pages(v) for v in vs]
    byt = 2 * n * H * d * 2
    try:
        us = timed(lambda j: trtllm_batch_decode_with_kv_cache(q, (kp[j], vp[j]), ws, bt, sl, n,
                                                                bmm1_scale=d ** -0.5), L)
        print(f"trtllm-gen decode n={n}: {us:.2f} us/layer  {byt / us / 1e3:.0f} GB/s")
    except Exception as e:
        print("trtllm-gen failed:", repr(e)[:300])
    kn = [k.transpose(0, 1) for k in ks]  # NHD views [n, H, d]
    vn = [v.transpose(0, 1) for v in vs]
    try:
        us = timed(lambda j: flashinfer.single_decode_with_kv_cache(q[0], kn[j], vn[j]), L)
        print(f"single_decode n={n}: {us:.2f} us/layer  {byt / us / 1e3:.0f} GB/s")
    except Exception as e:
        print("single_decode failed:", repr(e)[:300])
    del ks, vs, kp, vp, kn, vn
