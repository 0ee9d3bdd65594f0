"""Golden vectors for the measurement side (baselines + metrics), written by
the REAL reference (test infrastructure).

    python oracle/gen_golden_metrics.py   # in the build container (/root/reference present)

Covers engine.baseline_token_topk (engine.py:293-315),
engine.baseline_cluster_topk (:318-338), metrics.recovered_mass
(metrics.py:26-39), metrics.adaptive_token_budget (:41-50) and
metrics.cluster_approx_error (:61-76) on two small workloads, plus a cache
with duplicated key rows so top-k and the adaptive budget meet exact weight
ties (lower position wins).  Writes tests/golden/metrics_small.npz; the
workload tensors are stored too, so the fixture needs no reference at test
time.
"""
import os
import sys

import numpy as np

os.environ["DOUBLEP_KERNELS"] = "python"
sys.path.insert(0, "/root/reference/pkg/src")

from doublep import engine, metrics, workload  # noqa: E402
from doublep.clustering import build_clustered_cache  # noqa: E402
from doublep.kvcache import KvCache  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

TOKEN_BUDGETS = [1, 17, 200]
CLUSTER_BUDGETS = [1, 3, 9]
PS = [0.5, 0.9, 0.95, 0.99]
PLANS = [(0.95, 0.7), (0.9, 0.7)]


def record(rec, tag, cache, trace, cc, sink, window):
    rec[tag + "keys"] = cache.keys
    rec[tag + "values"] = cache.values
    rec[tag + "queries"] = trace.queries
    rec[tag + "sink_window"] = np.array([sink, window])
    L, Hq = cache.num_layers, trace.num_query_heads
    for s in range(trace.num_steps):
        for layer in range(L):
            for qh in range(Hq):
                h = qh // trace.gqa_group
                q = trace.query(s, layer, qh)
                pre = f"{tag}S{s}L{layer}Q{qh}_"
                for bud in TOKEN_BUDGETS + [cache.context_len]:
                    out, cap = engine.baseline_token_topk(q, cache, bud, layer, h)
                    w, _ = engine.full_attention_weights(q, cache, layer, h)
                    from doublep.selection import top_k_select
                    idx = top_k_select(w, bud)
                    rec[pre + f"tk{bud}_out"] = out.output
                    rec[pre + f"tk{bud}_cap"] = np.array(cap)
                    rec[pre + f"tk{bud}_norm"] = np.array(out.normalizer)
                    rec[pre + f"tk{bud}_set"] = np.sort(idx).astype(np.int32)
                for bud in CLUSTER_BUDGETS:
                    out = engine.baseline_cluster_topk(q, cache, cc, bud, layer, h)
                    rec[pre + f"ck{bud}_out"] = out.output
                for i, p in enumerate(PS):
                    rec[pre + f"ab{i}"] = np.array(metrics.adaptive_token_budget(q, cache, p, layer, h))
                for i, (p1, p2) in enumerate(PLANS):
                    cfg = engine.DoublePConfig(p1=p1, p2=p2, sink=sink, window=window)
                    _, plan, _ = engine.decode_step(q, cache, cc, cfg, layer, h)
                    rec[pre + f"rm{i}"] = np.array(metrics.recovered_mass(plan, q, cache))
                err, order = metrics.cluster_approx_error(q, cache, cc, layer, h)
                rec[pre + "cae_err"] = err
                rec[pre + "cae_order"] = order.astype(np.int32)


def main():
    rec = {}
    spec = workload.WorkloadSpec(context_len=640, head_dim=16, num_kv_heads=2, gqa_group=2, num_steps=1,
                                 tail_profile="mixed", seed=4)
    cache, trace = workload.generate(spec)
    cc = build_clustered_cache(cache, sink=spec.sink, window=spec.window, seed=0)
    record(rec, "A_", cache, trace, cc, spec.sink, spec.window)

    # exact ties: every key row duplicated (rows 2i and 2i+1 identical), so
    # weights tie in pairs and top-k must keep the lower position
    spec = workload.WorkloadSpec(context_len=512, head_dim=32, num_kv_heads=1, gqa_group=2, num_steps=1,
                                 tail_profile="peaked", seed=9)
    c0, trace = workload.generate(spec)
    k = np.repeat(c0.keys[:, :, ::2], 2, axis=2)
    v = c0.values.copy()
    cache = KvCache(keys=k, values=v)
    cc = build_clustered_cache(cache, sink=spec.sink, window=spec.window, seed=0)
    record(rec, "T_", cache, trace, cc, spec.sink, spec.window)

    path = os.path.join(OUT, "metrics_small.npz")
    np.savez_compressed(path, **rec)
    print("wrote", path, len(rec), "arrays")


if __name__ == "__main__":
    main()
