"""Time dp_select_global's three forms on a global log-mass table.

    python tools/gsel_probe.py [table.pt] [--iters 50]

table.pt: a [rows, ld] float64 table (bench.py --seq-shards ... with
DP_DUMP_GLM=path writes the 1M-token one); default: synthetic peaked rows.
Prints us per call (CUDA events, back to back) for the clustered one-launch
kernel (3), the split five-launch form (1) and one CTA per row (2), and
checks the three agree bit for bit."""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2602_05191_b200 import _native as N  # noqa: E402


def main():
    argv = sys.argv[1:]
    iters = 50
    if "--iters" in argv:
        k = argv.index("--iters")
        iters = int(argv[k + 1])
        argv = argv[:k] + argv[k + 2:]
    args = [a for a in argv if not a.startswith("--")]
    if args:
        lm = torch.load(args[0]).cuda()
    else:
        rng = np.random.default_rng(0)
        K = 32768
        rows = []
        for _ in range(32):
            b = rng.normal(0, 1, K) + np.log(rng.integers(1, 80, K))
            b[rng.integers(0, K, 300)] += rng.uniform(4, 14, 300)
            rows.append(b)
        lm = torch.from_numpy(np.stack(rows)).cuda()
    R, ld = lm.shape
    ks = torch.full((R,), ld, dtype=torch.int32, device="cuda")
    lib = N.lib()
    ws = torch.empty((lib.dp_select_global_workspace_bytes(R, ld),), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for path in (3, 1, 2):
        lib.dp_debug_set(11, path)
        st = torch.zeros((R, ld), dtype=torch.uint8, device="cuda")
        cnt = torch.zeros((R, 2), dtype=torch.int32, device="cuda")

        def call():
            N.check(lib.dp_select_global(N.ptr(lm), R, ld, N.ptr(ks), 0.95, 0.7, N.ptr(st), N.ptr(cnt), N.ptr(ws),
                                         ws.numel(), s))

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        res[path] = (st.clone(), cnt.clone())
        for dbg in ((0, 1, 2, 3, 4) if path == 3 and "--phases" in sys.argv else (0,)):
            lib.dp_debug_set(12, dbg)
            g = torch.cuda.CUDAGraph()  # device time only: the calls captured once, replayed
            with torch.cuda.graph(g):
                for _ in range(iters):
                    N.check(lib.dp_select_global(N.ptr(lm), R, ld, N.ptr(ks), 0.95, 0.7, N.ptr(st), N.ptr(cnt),
                                                 N.ptr(ws), ws.numel(), torch.cuda.current_stream().cuda_stream))
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            print(f"path {path} exit {dbg}: {e0.elapsed_time(e1) * 1000 / iters:8.2f} us per call (graph)")
        lib.dp_debug_set(12, 0)
    lib.dp_debug_set(11, 0)
    same = all(torch.equal(res[p][0], res[2][0]) and torch.equal(res[p][1], res[2][1]) for p in res)
    c = res[3][1].float()
    print(f"rows {R} ld {ld}; stage-1 kept mean {c[:, 0].mean():.0f}, stage-2 exact mean {c[:, 1].mean():.0f}; "
          f"paths identical: {same}")


if __name__ == "__main__":
    main()
