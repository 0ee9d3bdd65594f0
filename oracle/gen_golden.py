"""Generate golden vectors from the REAL reference package (test infrastructure).

Run in the build container, where ``/root/reference`` exists:

    python oracle/gen_golden.py

It imports ``doublep`` from ``/root/reference/pkg/src`` with the NumPy kernel
backend (``DOUBLEP_KERNELS=python``; the Cython extension is not built in the
read-only tree) and writes small ``.npz`` fixtures to ``tests/golden/``.  The
fixtures pin ``oracle/doublep_oracle.py`` (``tests/test_oracle_golden.py``)
and, through the oracle, the CUDA path.  Nothing on the GPU box reads
``/root/reference``; the fixtures travel instead.
"""

import hashlib
import os
import sys

import numpy as np

os.environ["DOUBLEP_KERNELS"] = "python"
sys.path.insert(0, "/root/reference/pkg/src")

from doublep import clustering, engine, workload  # noqa: E402
from doublep.clustering import build_clustered_cache  # noqa: E402
from doublep.engine import DoublePConfig, decode_step, full_attention  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

# (name, spec kwargs, (p1, p2) list, tokens_per_cluster)
CASES = [
    ("peaked_512_d16", dict(context_len=512, head_dim=16, num_kv_heads=2, gqa_group=2,
                            num_steps=2, tail_profile="peaked", seed=0), 32),
    ("mixed_1024_d32", dict(context_len=1024, head_dim=32, num_kv_heads=2, gqa_group=4,
                            num_steps=2, tail_profile="mixed", seed=3), 32),
    ("peaked_2048_d64", dict(context_len=2048, head_dim=64, num_kv_heads=1, gqa_group=4,
                             num_steps=2, tail_profile="peaked", seed=7), 32),
    ("heavy_1500_d128", dict(context_len=1500, head_dim=128, num_kv_heads=1, gqa_group=2,
                             num_steps=1, tail_profile="heavy", seed=11), 16),
    ("uniform_700_d16", dict(context_len=700, head_dim=16, num_kv_heads=1, gqa_group=2,
                             num_steps=1, tail_profile="uniform", seed=5), 32),
]
THRESHOLDS = [(0.95, 0.7), (0.99, 0.8), (0.9, 0.7), (1.0, 1.0), (0.5, 0.95)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    os.makedirs(OUT, exist_ok=True)
    manifest = []
    for name, kw, tpc in CASES:
        spec = workload.WorkloadSpec(**kw)
        cache, trace = workload.generate(spec)
        cc = build_clustered_cache(cache, sink=spec.sink, window=spec.window, seed=0,
                                   tokens_per_cluster=tpc)
        n = cache.context_len
        rec = {
            "keys_sha": np.array(sha(cache.keys)), "values_sha": np.array(sha(cache.values)),
            "queries_sha": np.array(sha(trace.queries)),
            "keys_probe": cache.keys[:, :, ::97, :3].copy(),
            "queries_probe": trace.queries[..., :3].copy(),
            "tokens_per_cluster": np.array(tpc),
        }
        L, H = cache.num_layers, cache.num_kv_heads
        for layer in range(L):
            for h in range(H):
                mid = n - spec.sink - spec.window
                k = clustering.default_cluster_count(mid, tpc)
                seed_h = int(np.random.SeedSequence([0, layer, h]).generate_state(1)[0])
                keys_mid = cache.keys[layer, h, spec.sink:n - spec.window]
                rng = np.random.default_rng(seed_h)
                init = clustering._plusplus_init(keys_mid.astype(np.float64), k, rng)
                fit = clustering.kmeans_fit(keys_mid, k, seed=seed_h)
                pre = f"L{layer}H{h}_"
                rec[pre + "init_centers"] = init
                rec[pre + "assign"] = fit.assignments.astype(np.int32)
                rec[pre + "objective"] = np.array(fit.objective)
                data = cc.estimation_data(layer, h)
                rec[pre + "centroids"] = data.centroids
                rec[pre + "value_means"] = data.value_means
                rec[pre + "sizes"] = np.array([c.size for c in data.clusters], np.int32)
        for ti, (p1, p2) in enumerate(THRESHOLDS):
            cfg = DoublePConfig(p1=p1, p2=p2, sink=spec.sink, window=spec.window)
            for s in range(trace.num_steps):
                for layer in range(L):
                    for qh in range(trace.num_query_heads):
                        h = qh // trace.gqa_group
                        q = trace.query(s, layer, qh)
                        out, plan, est = decode_step(q, cache, cc, cfg, layer, h)
                        pre = f"T{ti}S{s}L{layer}Q{qh}_"
                        rec[pre + "log_masses"] = est.log_masses
                        rec[pre + "stage1"] = plan.stage1.selected.astype(np.int32)
                        rec[pre + "cum1"] = np.array(plan.stage1.cumulative_mass)
                        rec[pre + "n_exact"] = np.array(plan.exact_clusters.size)
                        rec[pre + "n_tokens"] = np.array(plan.exact_tokens.size)
                        rec[pre + "tokens_sha"] = np.array(sha(plan.exact_tokens.astype(np.int64)))
                        rec[pre + "output"] = out.output
                        rec[pre + "normalizer"] = np.array(out.normalizer)
                        if ti == 0:
                            full = full_attention(q, cache, layer, h)
                            rec[pre + "full_output"] = full.output
                            rec[pre + "full_normalizer"] = np.array(full.normalizer)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        manifest.append(f"{name} {kw} tpc={tpc}")
        print("wrote", name)

    # decode-time growth: append 5 tokens then decode with p=(1,1) and (0.9,0.7)
    spec = workload.WorkloadSpec(context_len=300, head_dim=16, num_steps=1,
                                 tail_profile="peaked", seed=2)
    cache, trace = workload.generate(spec)
    cc = build_clustered_cache(cache, sink=4, window=64, seed=0)
    rng = np.random.default_rng(99)
    app_k = rng.normal(size=(5, 1, 1, 16)).astype(np.float32)
    app_v = rng.normal(size=(5, 1, 1, 16)).astype(np.float32)
    for t in range(5):
        cc.append_tokens(app_k[t], app_v[t])
    rec = {"app_k": app_k, "app_v": app_v}
    q = trace.query(0, 0, 0)
    for ti, (p1, p2) in enumerate([(1.0, 1.0), (0.9, 0.7)]):
        cfg = DoublePConfig(p1=p1, p2=p2)
        out, plan, est = decode_step(q, cache, cc, cfg, 0, 0)
        rec[f"T{ti}_output"] = out.output
        rec[f"T{ti}_stage1"] = plan.stage1.selected.astype(np.int32)
        rec[f"T{ti}_n_exact"] = np.array(plan.exact_clusters.size)
        rec[f"T{ti}_tokens"] = plan.exact_tokens.astype(np.int32)
        rec[f"T{ti}_normalizer"] = np.array(out.normalizer)
    rec["growth_full"] = engine.true_token_weights(q, cc, 0, 0)[0] @ cc.gather_values(
        0, 0, np.arange(cc.total_tokens)).astype(np.float64)
    np.savez_compressed(os.path.join(OUT, "growth_300_d16.npz"), **rec)
    manifest.append("growth_300_d16 peaked seed=2 append 5 (rng 99)")
    with open(os.path.join(OUT, "MANIFEST.txt"), "w") as f:
        f.write("# golden fixtures generated by oracle/gen_golden.py from /root/reference (doublep 0.1.0,"
                " DOUBLEP_KERNELS=python)\n")
        f.write(f"# thresholds (index T*): {THRESHOLDS}\n")
        f.write("\n".join(manifest) + "\n")


if __name__ == "__main__":
    main()
