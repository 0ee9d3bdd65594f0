"""Randomised parity sweep of the fused decode path against the CPU oracle
(the §8c protocol of tests/test_gpu_parity.py, over many random geometries).

    python tools/parity_sweep.py [cases] [seed] [max_context]

Each case draws (context, kv heads, G, head dim, dtype, tail profile, p1, p2,
plan cluster size), builds the workload with the reference generator law,
clusters it on the GPU, runs sparse_attention through the C ABI and checks
every q head: log-masses vs the oracle fed the GPU's tables, the two
selection stages (exact / order tie / threshold tie / real), and the output
error when both stages match.  Prints one summary line per case and a total.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import doublep_oracle as O  # noqa: E402
from parity import classify_sets, oracle_tables  # noqa: E402

from paper_2602_05191_b200 import _native as N  # noqa: E402
from paper_2602_05191_b200 import cluster_layer, sparse_attention  # noqa: E402

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-3}


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1234)
    nmax = int(sys.argv[3]) if len(sys.argv) > 3 else 40000
    sizes = [x for x in (300, 700, 1500, 3000, 6000, 12000, 24000, 40000, 80000, 131072) if x <= nmax]
    totals = {"heads": 0, "exact": 0, "order_tie": 0, "threshold_tie": 0, "real": 0, "out_checked": 0,
              "out_fail": 0, "lm_fail": 0}
    worst = {torch.float32: 0.0, torch.bfloat16: 0.0}
    t0 = time.time()
    for c in range(cases):
        n = int(rng.choice(sizes))
        H = int(rng.choice([1, 2, 3]))
        G = int(rng.choice([1, 2, 3, 4, 6, 8]))
        d = int(rng.choice([32, 64, 128, 128]))
        dtype = torch.bfloat16 if rng.random() < 0.6 else torch.float32
        prof = str(rng.choice(["peaked", "mixed", "heavy", "uniform"]))
        p1 = float(rng.choice([0.5, 0.8, 0.9, 0.95, 0.99, 1.0]))
        p2 = float(rng.choice([0.3, 0.7, 0.8, 0.95, 1.0]))
        cl = int(rng.choice([0, 0, 4, 8, 12, 16]))
        seed = int(rng.integers(1 << 30))
        B = int(rng.choice([1, 1, 2, 3]))
        qdt = torch.float32 if rng.random() < 0.3 else dtype  # fp32 queries over bf16 caches too
        ks, vs, qs = [], [], []
        for b in range(B):
            spec = O.WorkloadSpec(context_len=n, head_dim=d, num_kv_heads=H, gqa_group=G, num_steps=1,
                                  tail_profile=prof, seed=seed + b)
            keys, values, queries = O.generate(spec)
            ks.append(keys[0])
            vs.append(values[0])
            qs.append(queries[0, 0])
        kd = torch.from_numpy(np.ascontiguousarray(np.stack(ks))).cuda().to(dtype)
        vd = torch.from_numpy(np.ascontiguousarray(np.stack(vs))).cuda().to(dtype)
        q = torch.from_numpy(np.ascontiguousarray(np.stack(qs))).cuda().to(dtype).to(qdt)
        N.lib().dp_debug_set(1, cl if cl >= G else 0)
        tag = (f"case {c:3d}: B={B} n={n:5d} H={H} G={G} d={d:3d} {str(dtype)[6:]:8s} q {str(qdt)[6:]:8s} "
               f"{prof:7s} p=({p1},{p2}) cl={cl or 'auto'}")
        layer = cluster_layer(kd, vd, fp64_assign=False)
        try:
            out, ws = sparse_attention(q, layer, p1, p2, return_plan=True)
        except Exception as e:  # noqa: BLE001
            totals.setdefault("errors", []).append(tag)
            print(tag + f": ERROR {e} (K={layer.nclusters.tolist()}, cap={layer.cluster_cap})", flush=True)
            continue
        outs = out.double().cpu().numpy()
        lms = ws.log_mass.cpu().numpy()
        sts = ws.state.cpu().numpy()
        cls = {}
        for b, hq in [(b, hq) for b in range(B) for hq in range(H * G)]:
            out, lm, st = outs[b], lms[b], sts[b]
            kf = kd[b].double().cpu().numpy()
            vf = vd[b].double().cpu().numpy()
            h = hq // G
            t = oracle_tables(layer, b, h)
            o_out, o_plan, o_est = O.decode_step(q[b, hq].double().cpu().numpy(), kf[h], vf[h], t, p1, p2,
                                                 layer.sink, layer.window)
            K = len(t.members)
            if K and np.max(np.abs(lm[hq, :K] - o_est.log_masses)) > 1e-9:
                totals["lm_fail"] += 1
            c1, c2 = classify_sets(o_est, o_plan, st[hq], p1, p2) if K else ("exact", "exact")
            for x in (c1, c2):
                totals[x] += 1
                cls[x] = cls.get(x, 0) + 1
            totals["heads"] += 1
            if c1 == "exact" and c2 == "exact":
                totals["out_checked"] += 1
                err = O.output_error(out[hq], o_out.output)
                worst[dtype] = max(worst[dtype], err)
                if err > TOL[dtype]:
                    totals["out_fail"] += 1
        print(f"{tag}: {cls}", flush=True)
    N.lib().dp_debug_set(1, 0)
    print(f"TOTAL over {cases} cases, {totals['heads']} q heads ({time.time() - t0:.0f}s): {totals}")
    print("worst output rel-L2 error: fp32 %.2e (tol 1e-5), bf16 %.2e (tol 2e-3)" %
          (worst[torch.float32], worst[torch.bfloat16]))
    ok = totals["real"] == 0 and totals["out_fail"] == 0 and totals["lm_fail"] == 0 and not totals.get("errors")
    print("PASS" if ok else "FAIL")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
