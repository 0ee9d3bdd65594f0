"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same seeded inputs.  Tolerances (BASELINE.json
north_star): selection bit-exact except score ties within 1e-6; outputs
rel-L2 <= 1e-5 (fp32 cache) / 2e-3 (bf16 cache)."""

import math

import numpy as np
import pytest
import torch

from oracle import doublep_oracle as O
from parity import classify_sets, compare_plan, oracle_tables

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-3}


def _workload(n, d, H, G, profile, seed, steps=1):
    spec = O.WorkloadSpec(context_len=n, head_dim=d, num_kv_heads=H, gqa_group=G, num_steps=steps,
                          tail_profile=profile, seed=seed)
    return spec, *O.generate(spec)


def _to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)


def _layer(keys, values, dtype, **kw):
    from paper_2602_05191_b200 import cluster_layer

    k = _to_dev(keys[0], dtype).unsqueeze(0)  # [1,H,N,d]
    v = _to_dev(values[0], dtype).unsqueeze(0)
    return cluster_layer(k, v, **kw), k, v


def _check_decode(layer, kdev, vdev, queries, G, p1, p2, dtype, counts=None):
    """Batched product path vs the oracle fed the GPU's tables."""
    from paper_2602_05191_b200 import sparse_attention

    H = layer.kv_heads
    q = _to_dev(queries, dtype).unsqueeze(0)  # [1,Hq,d]
    out, ws = sparse_attention(q, layer, p1, p2, return_plan=True)
    out = out[0].double().cpu().numpy()
    lse = ws.lse[0].double().cpu().numpy()
    lm_g = ws.log_mass[0].cpu().numpy()
    cnt = ws.counts[0].cpu().numpy()
    # full descending order from a debug select over the same log-masses
    from paper_2602_05191_b200 import _native as N

    order = torch.zeros_like(ws.state, dtype=torch.int32)
    st2 = torch.zeros_like(ws.state)
    c2 = torch.zeros_like(ws.counts)
    N.check(N.lib().dp_select(layer.view(), G, p1, p2, N.ptr(ws.log_mass), N.ptr(st2), N.ptr(c2),
                              N.ptr(order), None, None, None, 0, torch.cuda.current_stream().cuda_stream))
    order = order[0].cpu().numpy()
    st_plan = ws.state[0].cpu().numpy()  # the fused plan kernel's selection
    classes = {}
    kf = kdev[0].double().cpu().numpy()  # exact upcast of what the GPU read
    vf = vdev[0].double().cpu().numpy()
    for hq in range(H * G):
        h = hq // G
        t = oracle_tables(layer, 0, h)
        qv = q[0, hq].double().cpu().numpy()
        o_out, o_plan, o_est = O.decode_step(qv, kf[h], vf[h], t, p1, p2, layer.sink, layer.window)
        K = len(t.members)
        np.testing.assert_allclose(lm_g[hq, :K], o_est.log_masses, rtol=0, atol=1e-9)
        c1, c2_ = classify_sets(o_est, o_plan, st_plan[hq], p1, p2)
        # the debug (full bitonic sort) select must agree with the oracle too
        d1, d2 = compare_plan(o_est, o_plan, order[hq], int(c2[0, hq, 0]), int(c2[0, hq, 1]), p1, p2)
        assert d1 != "real" and d2 != "real", (hq, d1, d2)
        assert int(cnt[hq, 0]) == int((st_plan[hq, :K] >= 1).sum()) and int(cnt[hq, 1]) == int((st_plan[hq, :K] == 2).sum())
        classes[c1] = classes.get(c1, 0) + 1
        classes[c2_] = classes.get(c2_, 0) + 1
        assert c1 != "real" and c2_ != "real", (hq, c1, c2_)
        if c1 == "exact" and c2_ == "exact":
            err = O.output_error(out[hq], o_out.output)
            assert err <= TOL[dtype], (hq, err)
            assert abs(lse[hq] - o_out.log_normalizer) <= 1e-4 * max(1.0, abs(o_out.log_normalizer))
    if counts is not None:
        counts.update(classes)
    return classes


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("profile,n,d,H,G,seed", [
    ("peaked", 2048, 128, 2, 4, 0),
    ("mixed", 1536, 64, 2, 4, 1),
    ("heavy", 1024, 128, 1, 8, 2),
    ("uniform", 700, 32, 1, 2, 3),
])
def test_decode_parity(dtype, profile, n, d, H, G, seed):
    spec, keys, values, queries = _workload(n, d, H, G, profile, seed, steps=2)
    layer, kd, vd = _layer(keys, values, dtype)
    # (1.0, 0.7) and (0.8, 1.0): the clamped stage 1 with a real stage-2 cut, and a
    # stage 2 that keeps the whole retained set (select.cuh's p >= 1 branches)
    for p1, p2 in [(0.95, 0.7), (0.99, 0.8), (0.9, 0.7), (1.0, 1.0), (0.5, 0.95), (1.0, 0.7), (0.8, 1.0)]:
        for s in range(2):
            _check_decode(layer, layer_rows(kd), layer_rows(vd), queries[s, 0], G, p1, p2, dtype)


def layer_rows(t):
    return t  # position-ordered source rows [1,H,N,d]


def test_dense_parity():
    from paper_2602_05191_b200 import dense_attention

    for dtype in (torch.float32, torch.bfloat16):
        spec, keys, values, queries = _workload(3000, 128, 2, 4, "peaked", 5)
        layer, kd, vd = _layer(keys, values, dtype)
        q = _to_dev(queries[0, 0], dtype).unsqueeze(0)
        out, lse = dense_attention(q, layer, return_lse=True)
        kf = kd[0].double().cpu().numpy()
        vf = vd[0].double().cpu().numpy()
        for hq in range(8):
            ref = O.full_attention(q[0, hq].double().cpu().numpy(), kf[hq // 4], vf[hq // 4])
            assert O.output_error(out[0, hq].double().cpu().numpy(), ref.output) <= TOL[dtype]
            assert abs(float(lse[0, hq]) - ref.log_normalizer) <= 1e-4 * abs(ref.log_normalizer) + 1e-5


def test_kmeanspp_picks_exact():
    """dp_kmeanspp replays the reference's k-means++ picks bit-exactly."""
    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200.cache import head_seed, rng_stream

    spec, keys, values, _ = _workload(4096, 64, 2, 1, "peaked", 7)
    n, sink, window = 4096, 4, 64
    M = n - sink - window
    k = O.default_cluster_count(M)
    for dtype in (torch.float32, torch.bfloat16):
        kd = _to_dev(keys[0], dtype).unsqueeze(0)
        p = N.ClusterParams()
        p.batch, p.kv_heads, p.head_dim, p.dtype = 1, 2, 64, 0 if dtype == torch.float32 else 1
        p.n_tokens, p.sink, p.window, p.k, p.max_iters, p.fp64_assign = n, sink, window, k, 25, 1
        firsts, us = [], []
        for h in range(2):
            f, u, _ = rng_stream(head_seed(0, 0, h), M, k)
            firsts.append(f)
            us.append(u)
        f_d = torch.tensor(firsts, dtype=torch.int32, device="cuda")
        u_d = torch.from_numpy(np.stack(us)).cuda()
        picks = torch.zeros((2, k), dtype=torch.int32, device="cuda")
        ws = torch.empty((N.lib().dp_cluster_workspace_bytes(p),), dtype=torch.uint8, device="cuda")
        N.check(N.lib().dp_kmeanspp(p, N.ptr(kd), N.ptr(f_d), N.ptr(u_d), None, None, N.ptr(picks),
                                    N.ptr(ws), ws.numel(), torch.cuda.current_stream().cuda_stream))
        kf = kd[0].double().cpu().numpy()
        for h in range(2):
            mid = kf[h, sink:n - window]
            _, want = O.plusplus_init(mid, k, np.random.default_rng(head_seed(0, 0, h)))
            np.testing.assert_array_equal(picks[h].cpu().numpy(), want)


@pytest.mark.parametrize("fp64", [True, False])
def test_cluster_build_parity(fp64):
    """Clustering parity: same init, assignment
    agreement >= 1 - 1e-3, objective within 1e-5 (exact in fp64 mode)."""
    spec, keys, values, _ = _workload(3072, 64, 2, 1, "mixed", 9)
    n, sink, window = 3072, 4, 64
    layer, kd, vd = _layer(keys, values, torch.float32, fp64_assign=fp64)
    k = O.default_cluster_count(n - sink - window)
    for h in range(2):
        t_o, fit = O.build_head_tables(keys[0, h], values[0, h], k, sink, window,
                                       seed_for_head=O.head_seed(0, 0, h))
        t_g = layer.head_tables(0, h)
        lab_o = np.full(n, -1)
        lab_g = np.full(n, -1)
        for c, m in enumerate(t_o.members):
            lab_o[m] = c
        for c, m in enumerate(t_g["members"]):
            lab_g[m] = c
        agree = np.mean(lab_o[sink:n - window] == lab_g[sink:n - window])
        obj_g = layer.objective[h, : int(layer.iters[h])].cpu().numpy()
        if fp64:
            assert agree == 1.0
            np.testing.assert_allclose(obj_g, fit.objective, rtol=1e-10)
            np.testing.assert_allclose(t_g["centroids"], t_o.centroids, rtol=0, atol=1e-6)
            np.testing.assert_allclose(t_g["value_means"], t_o.value_means, rtol=0, atol=1e-6)
        else:
            assert agree >= 1 - 1e-3
            assert abs(obj_g[-1] - fit.objective[-1]) <= 1e-5 * fit.objective[-1]
        # partition + contiguity invariants (SPEC.md: partition property)
        allm = np.sort(np.concatenate(t_g["members"]))
        np.testing.assert_array_equal(allm, np.arange(sink, n - window))
        rows = layer.keys[0, h].float().cpu().numpy()
        perm = layer.perm[0, h].cpu().numpy()
        np.testing.assert_array_equal(rows[: n], keys[0, h][perm[:n]])


@pytest.mark.parametrize("d", [64, 128])
def test_cluster_build_parity_tensor_cores(d):
    """Lloyd assignment on tcgen05 (bf16 keys exact, centroids as three bf16
    terms, fp32 TMEM accumulation) against the oracle on the same bf16 keys:
    assignment agreement >= 1 - 1e-3, final objective within 1e-5."""
    spec, keys, values, _ = _workload(3072, d, 2, 1, "mixed", 9)
    n, sink, window = 3072, 4, 64
    kb = torch.from_numpy(keys[0]).to(torch.bfloat16)
    keys_b = kb.double().numpy()[None]  # the values the GPU clusters (exact upcast)
    layer, kd, vd = _layer(keys_b, values, torch.bfloat16, fp64_assign=False, tensor_cores=True)
    k = O.default_cluster_count(n - sink - window)
    for h in range(2):
        t_o, fit = O.build_head_tables(keys_b[0, h], values[0, h], k, sink, window,
                                       seed_for_head=O.head_seed(0, 0, h))
        t_g = layer.head_tables(0, h)
        lab_o = np.full(n, -1)
        lab_g = np.full(n, -1)
        for c, m in enumerate(t_o.members):
            lab_o[m] = c
        for c, m in enumerate(t_g["members"]):
            lab_g[m] = c
        agree = np.mean(lab_o[sink:n - window] == lab_g[sink:n - window])
        obj_g = layer.objective[h, : int(layer.iters[h])].cpu().numpy()
        assert agree >= 1 - 1e-3, agree
        assert abs(obj_g[-1] - fit.objective[-1]) <= 1e-5 * fit.objective[-1]
        allm = np.sort(np.concatenate(t_g["members"]))
        np.testing.assert_array_equal(allm, np.arange(sink, n - window))


def _gpu_order(layer, ws, G, p1, p2):
    """Full descending order from a debug dp_select over the same log-masses."""
    from paper_2602_05191_b200 import _native as N

    order = torch.zeros_like(ws.state, dtype=torch.int32)
    st2 = torch.zeros_like(ws.state)
    c2 = torch.zeros_like(ws.counts)
    N.check(N.lib().dp_select(layer.view(), G, p1, p2, N.ptr(ws.log_mass), N.ptr(st2), N.ptr(c2),
                              N.ptr(order), None, None, None, 0, torch.cuda.current_stream().cuda_stream))
    return order[0].cpu().numpy()


def test_golden_end_to_end():
    """GPU clustering + decode against the real reference's golden outputs
    (reference centroids are fp64, the device's fp32: selection compared
    under the tie protocol, outputs within the fp32 bar)."""
    import os

    from conftest import GOLDEN
    from paper_2602_05191_b200 import sparse_attention
    from parity import classify_stage

    g = np.load(os.path.join(GOLDEN, "peaked_2048_d64.npz"))
    spec, keys, values, queries = _workload(2048, 64, 1, 4, "peaked", 7, steps=2)
    layer, kd, vd = _layer(keys, values, torch.float32)
    np.testing.assert_array_equal(layer.head_tables(0, 0)["sizes"], g["L0H0_sizes"])
    np.testing.assert_allclose(layer.head_tables(0, 0)["centroids"], g["L0H0_centroids"], atol=1e-6)
    ties = 0
    for ti, (p1, p2) in enumerate([(0.95, 0.7), (0.99, 0.8), (0.9, 0.7), (1.0, 1.0), (0.5, 0.95)]):
        for s in range(2):
            q = _to_dev(queries[s, 0], torch.float32).unsqueeze(0)
            out, ws = sparse_attention(q, layer, p1, p2, return_plan=True)
            order = _gpu_order(layer, ws, 4, p1, p2)
            for hq in range(4):
                pre = f"T{ti}S{s}L0Q{hq}_"
                lm = g[pre + "log_masses"]
                probs = O.softmax(lm)
                order_o = np.argsort(-probs, kind="stable")
                cum = np.cumsum(probs[order_o]) / probs.sum()
                n1o = g[pre + "stage1"].size
                np.testing.assert_array_equal(order_o[:n1o], g[pre + "stage1"])
                c1 = classify_stage(probs, order_o, n1o, order[hq], int(ws.counts[0, hq, 0]), cum, p1)
                assert c1 != "real", (ti, s, hq)
                if c1 != "exact":
                    ties += 1
                    continue
                n2o = int(g[pre + "n_exact"])
                sub = probs[order_o[:n1o]]
                c2 = classify_stage(probs, order_o, n2o, order[hq], int(ws.counts[0, hq, 1]),
                                    np.cumsum(sub) / sub.sum(), p2)
                assert c2 != "real", (ti, s, hq)
                if c2 != "exact":
                    ties += 1
                    continue
                err = O.output_error(out[0, hq].double().cpu().numpy(), g[pre + "output"])
                assert err <= 1e-5, err
    assert ties <= 8  # p = 1.0 threshold ties (cumsum/total reaches 1 early)


def test_reference_semantics_on_gpu():
    """Reference unit-test semantics through the reference-signature API."""
    import paper_2602_05191_b200 as dp

    rng = np.random.default_rng(0)
    # exactness collapse with singleton clusters (test_engine.py:128-136)
    keys = rng.normal(size=(1, 1, 40, 8)).astype(np.float32)
    vals = rng.normal(size=(1, 1, 40, 8)).astype(np.float32)
    cache = dp.KvCache(keys, vals)
    cc = dp.build_clustered_cache(cache, k=40, sink=0, window=0)
    cfg = dp.DoublePConfig(p1=1.0, p2=1.0, sink=0, window=0)
    q = rng.normal(size=8).astype(np.float32)
    out, plan, est = dp.decode_step(q, cache, cc, cfg, 0, 0)
    ref = O.full_attention(q.astype(np.float64), keys[0, 0].astype(np.float64), vals[0, 0].astype(np.float64))
    assert O.output_error(out.output, ref.output) <= 1e-5
    assert out.normalizer == pytest.approx(ref.normalizer, rel=1e-5)
    # two-token cluster mass 2e vs 1+e^2 (test_engine.py:113-125), embedded in
    # d=16 so the logits {0, 2} stay exact (sqrt(16) = 4)
    k2 = np.zeros((1, 1, 2, 16), np.float32)
    k2[0, 0, 1, 0] = 8.0
    cache2 = dp.KvCache(k2, np.ones((1, 1, 2, 16), np.float32))
    cc2 = dp.build_clustered_cache(cache2, k=1, sink=0, window=0)
    q2 = np.zeros(16, np.float32)
    q2[0] = 1.0
    est2 = dp.estimate_cluster_distribution(q2, cc2, 0, 0)
    assert math.exp(est2.log_masses[0]) == pytest.approx(2 * math.e, rel=1e-9)
    # mixture weights sum to one (test_engine.py:151-159)
    keys3 = rng.normal(size=(1, 1, 128, 8)).astype(np.float32)
    cache3 = dp.KvCache(keys3, np.ones((1, 1, 128, 8), np.float32))
    cc3 = dp.build_clustered_cache(cache3, k=9, sink=2, window=16)
    cfg3 = dp.DoublePConfig(p1=0.9, p2=0.6, sink=2, window=16)
    out3, plan3, _ = dp.decode_step(rng.normal(size=8).astype(np.float32) * 2, cache3, cc3, cfg3, 0, 0)
    np.testing.assert_allclose(out3.output, np.ones(8), atol=1e-6)
    assert out3.approx_cluster_count == plan3.approx_clusters.size
    # p1 = p2 = 1 keeps everything (test_engine.py:115-123)
    plan4 = dp.plan_selection(dp.estimate_cluster_distribution(q, cc3 if False else cc, 0, 0), cfg)
    assert plan4.approx_clusters.size == 0 and plan4.exact_tokens.size == 40
    # error messages
    with pytest.raises(ValueError, match="config/cache mismatch"):
        dp.decode_step(q, cache, cc, dp.DoublePConfig(0.9, 0.7, sink=4, window=0), 0, 0)
    other = dp.KvCache(keys, vals)
    with pytest.raises(ValueError, match="mismatch"):
        dp.sparse_attention(q, other, cc, plan, 0, 0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        dp.full_attention(np.ones(5, np.float32), cache, 0, 0)


def test_growth_parity():
    """append_tokens on the device vs the oracle's residual singleton pool."""
    import paper_2602_05191_b200 as dp

    spec, keys, values, queries = _workload(300, 16, 1, 1, "peaked", 2)
    cache = dp.KvCache(keys, values)
    cc = dp.build_clustered_cache(cache, sink=4, window=64, growth=8)
    rng = np.random.default_rng(99)
    app_k = rng.normal(size=(5, 1, 1, 16)).astype(np.float32)
    app_v = rng.normal(size=(5, 1, 1, 16)).astype(np.float32)
    for t in range(5):
        cc.append_tokens(app_k[t], app_v[t])
    assert cc.total_tokens == 305
    base = oracle_tables(cc.layers[0], 0, 0)
    # the first layer's tables already include the residuals; rebuild the base
    kprefill = int(cc.layers[0]._prefill_k)
    base = O.HeadTables(members=base.members[:kprefill], centroids=base.centroids[:kprefill],
                        value_means=base.value_means[:kprefill])
    kf = np.concatenate([keys[0, 0], app_k[:, 0, 0]]).astype(np.float64)
    vf = np.concatenate([values[0, 0], app_v[:, 0, 0]]).astype(np.float64)
    t = O.grow_tables(base, kf, vf, 300, 305, 64)
    q = queries[0, 0, 0]
    for p1, p2 in [(1.0, 1.0), (0.9, 0.7)]:
        out, plan, _ = dp.decode_step(q, cache, cc, dp.DoublePConfig(p1, p2), 0, 0)
        o_out, o_plan, _ = O.decode_step(q.astype(np.float64), kf, vf, t, p1, p2, 4, 64)
        np.testing.assert_array_equal(plan.stage1.selected, o_plan.stage1.selected)
        np.testing.assert_array_equal(plan.exact_tokens, o_plan.exact_tokens)
        assert O.output_error(out.output, o_out.output) <= 1e-5


@pytest.mark.parametrize("cl", [4, 8, 10, 12, 16])
def test_plan_cluster_sizes_and_multi_tile(cl):
    """The fused plan at both cluster sizes, with slices longer than one
    128-row centroid tile (n = 40K -> ~1250 clusters)."""
    from paper_2602_05191_b200 import _native as N

    N.lib().dp_debug_set(1, cl)
    try:
        spec, keys, values, queries = _workload(40000, 128, 1, 4, "peaked", 11)
        layer, kd, vd = _layer(keys, values, torch.bfloat16, fp64_assign=False)
        for p1, p2 in [(0.95, 0.7), (0.99, 0.8)]:
            _check_decode(layer, kd, vd, queries[0, 0], 4, p1, p2, torch.bfloat16)
    finally:
        N.lib().dp_debug_set(1, 0)


def test_full_size_exact_collapse_matches_dense():
    """Size-independent property at the bench shape (32K, 8 kv heads, G=4):
    with p1 = p2 = 1 every cluster is exact, so the sparse step must equal the
    dense kernel (engine.py:128-136 exactness collapse)."""
    from paper_2602_05191_b200 import cluster_layer, dense_attention, sparse_attention
    from paper_2602_05191_b200.workload import generate_layer, generate_queries

    k, v, c = generate_layer(1, 8, 32768, 128)
    layer = cluster_layer(k, v, fp64_assign=False)
    q = torch.from_numpy(generate_queries(c, 4, 1)[0]).cuda().to(torch.bfloat16)
    sp = sparse_attention(q, layer, 1.0, 1.0).clone()
    de = dense_attention(q, layer).clone()
    err = ((sp - de).norm(dim=-1) / de.norm(dim=-1)).max().item()
    assert err <= 2e-3, err
    # and at the default thresholds the kept mass is large: the output stays close to dense
    sp95 = sparse_attention(q, layer, 0.95, 0.7).clone()
    assert torch.isfinite(sp95).all()


def test_sequence_sharded_merge_on_gpu():
    """Config-5 exchange math on one GPU: two sequence shards, dense attention
    per shard (kernel lse), LSE merge == dense attention over all tokens."""
    from paper_2602_05191_b200 import cluster_layer, dense_attention
    from paper_2602_05191_b200.sharding import lse_merge

    spec, keys, values, queries = _workload(4096, 128, 2, 4, "peaked", 7)
    kd = _to_dev(keys[0], torch.bfloat16).unsqueeze(0)
    vd = _to_dev(values[0], torch.bfloat16).unsqueeze(0)
    q = _to_dev(queries[0, 0], torch.bfloat16).unsqueeze(0)
    full = cluster_layer(kd, vd, fp64_assign=False)
    ref = dense_attention(q, full).clone()
    half = 2048
    a = cluster_layer(kd[:, :, :half].contiguous(), vd[:, :, :half].contiguous(), fp64_assign=False, window=0)
    b = cluster_layer(kd[:, :, half:].contiguous(), vd[:, :, half:].contiguous(), fp64_assign=False, sink=0)
    oa, la = dense_attention(q, a, return_lse=True)
    oa, la = oa.clone(), la.clone()
    ob, lb = dense_attention(q, b, return_lse=True)
    out, _ = lse_merge(torch.stack([oa, ob.clone()]), torch.stack([la, lb.clone()]))
    err = ((out - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
    assert err <= 1e-4, err


@pytest.mark.parametrize("budget", [1, 7, 40])
def test_cluster_topk_baseline_parity(budget):
    """GPU fixed cluster-budget baseline (engine.py:318-338) vs the oracle fed
    the GPU's tables."""
    from paper_2602_05191_b200 import cluster_topk_attention

    spec, keys, values, queries = _workload(2048, 128, 2, 4, "peaked", 13)
    for dtype in (torch.float32, torch.bfloat16):
        layer, kd, vd = _layer(keys, values, dtype)
        q = _to_dev(queries[0, 0], dtype).unsqueeze(0)
        out, ws = cluster_topk_attention(q, layer, budget, return_plan=True)
        out = out[0].double().cpu().numpy()
        kf = kd[0].double().cpu().numpy()
        vf = vd[0].double().cpu().numpy()
        for hq in range(8):
            h = hq // 4
            t = oracle_tables(layer, 0, h)
            K = len(t.members)
            ref = O.cluster_topk(q[0, hq].double().cpu().numpy(), kf[h], vf[h], t, min(budget, K), layer.sink,
                                 layer.window)
            assert int(ws.counts[0, hq, 1]) == min(budget, K)
            assert O.output_error(out[hq], ref.output) <= TOL[dtype], (hq, budget)


@pytest.mark.parametrize("G", [3, 4])
def test_batched_sequences_parity(G):
    """Batch > 1 (config 3 layout): two sequences with different caches in one
    layer, one decode step; every (sequence, q head) against the oracle fed
    that sequence's GPU tables.  G = 3 exercises a non-power-of-two group."""
    from paper_2602_05191_b200 import cluster_layer, sparse_attention

    B, H, n, d = 2, 2, 1500, 128
    ks, vs, qs = [], [], []
    for b in range(B):
        spec, keys, values, queries = _workload(n, d, H, G, "peaked", 20 + b)
        ks.append(keys[0])
        vs.append(values[0])
        qs.append(queries[0, 0])
    kd = _to_dev(np.stack(ks), torch.bfloat16)  # [B,H,N,d]
    vd = _to_dev(np.stack(vs), torch.bfloat16)
    q = _to_dev(np.stack(qs), torch.bfloat16)    # [B,Hq,d]
    layer = cluster_layer(kd, vd, fp64_assign=False)
    out, ws = sparse_attention(q, layer, 0.95, 0.7, return_plan=True)
    out = out.double().cpu().numpy()
    st = ws.state.cpu().numpy()
    for b in range(B):
        kf = kd[b].double().cpu().numpy()
        vf = vd[b].double().cpu().numpy()
        for hq in range(H * G):
            h = hq // G
            t = oracle_tables(layer, b, h)
            o_out, o_plan, o_est = O.decode_step(q[b, hq].double().cpu().numpy(), kf[h], vf[h], t, 0.95, 0.7,
                                                 layer.sink, layer.window)
            c1, c2 = classify_sets(o_est, o_plan, st[b, hq], 0.95, 0.7)
            assert c1 != "real" and c2 != "real", (b, hq, c1, c2)
            if c1 == "exact" and c2 == "exact":
                assert O.output_error(out[b, hq], o_out.output) <= TOL[torch.bfloat16], (b, hq)


def test_decode_graph_matches_eager():
    """DecodeGraph (the step's per-layer sparse_attention calls captured as one
    CUDA graph, shared workspace) reproduces the eager calls layer by layer."""
    from paper_2602_05191_b200 import DecodeGraph, DecodeWorkspace, cluster_layer, sparse_attention
    from paper_2602_05191_b200.workload import generate_layer, generate_queries

    L, H, G, n, d = 3, 2, 4, 4096, 128
    layers, qs = [], []
    for li in range(L):
        k, v, c = generate_layer(1, H, n, d, layer=li)
        layers.append(cluster_layer(k, v, fp64_assign=False, layer=li))
        qs.append(torch.from_numpy(generate_queries(c, G, 1, layer=li)[0]).cuda().to(torch.bfloat16))
    q = torch.stack(qs)  # [L, 1, Hq, d]
    ws = DecodeWorkspace(layers[0], G)
    want = torch.stack([sparse_attention(q[li], layers[li], 0.95, 0.7, workspace=ws).clone() for li in range(L)])
    dg = DecodeGraph(layers, q.clone(), 0.95, 0.7, workspace=ws)
    for _ in range(2):
        got = dg.replay()
        torch.cuda.synchronize()
        err = ((got - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
        assert err <= 1e-5, err
    # pinned host buffers inside the graph: q in, every layer's output out
    hq = q.cpu().pin_memory()
    ho = torch.zeros(q.shape, dtype=torch.float32).pin_memory()
    qbuf = torch.zeros_like(q)
    dg2 = DecodeGraph(layers, qbuf, 0.95, 0.7, workspace=ws, host_q=hq, host_out=ho)
    ho.zero_()
    got = dg2.replay()
    torch.cuda.synchronize()
    assert got.data_ptr() == ho.data_ptr()
    err = ((got - want.cpu()).norm(dim=-1) / want.cpu().norm(dim=-1)).max().item()
    assert err <= 1e-5, err


def test_nonfinite_query_does_not_fault():
    """A NaN/Inf query (garbage in an uninitialised buffer) gives garbage
    outputs but must not fault the plan or attention kernels."""
    from paper_2602_05191_b200 import DecodeWorkspace, cluster_layer, sparse_attention
    from paper_2602_05191_b200.workload import generate_layer

    k, v, _ = generate_layer(1, 2, 4096, 128)
    lay = cluster_layer(k, v, fp64_assign=False)
    ws = DecodeWorkspace(lay, 4)
    for bad in (float("nan"), float("inf"), -float("inf")):
        q = torch.full((1, 8, 128), bad, dtype=torch.bfloat16, device="cuda")
        sparse_attention(q, lay, 0.95, 0.7, workspace=ws)
        torch.cuda.synchronize()
    q = torch.randn((1, 8, 128), device="cuda").to(torch.bfloat16)
    out = sparse_attention(q, lay, 0.95, 0.7, workspace=ws)  # the workspace is still usable
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()


def test_tensor_core_assign_tiny_tables():
    """Tensor-core assignment with fewer than 128 centroid rows in the whole
    split table (3 * B*H * k < 128): the TMA boxes must still complete (this
    shape used to hang) and the result equals the fp64 path."""
    from paper_2602_05191_b200 import cluster_layer
    from paper_2602_05191_b200.workload import generate_layer

    k, v, _ = generate_layer(2, 1, 700, 128)  # B=2, H=1, 20 clusters per head -> 120 split rows
    tc = cluster_layer(k, v, fp64_assign=False, tensor_cores=True)
    ref = cluster_layer(k, v, fp64_assign=True)
    torch.cuda.synchronize()
    assert torch.equal(tc.offs, ref.offs) and torch.equal(tc.perm, ref.perm)


def test_nonfinite_query_other_entry_points():
    """The unfused score/select/attend path, the cluster top-k baseline and the
    measurement kernels also survive a NaN query (garbage out, no fault)."""
    from paper_2602_05191_b200 import cluster_layer, cluster_topk_attention
    from paper_2602_05191_b200 import metrics as M
    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200.workload import generate_layer

    k, v, _ = generate_layer(1, 2, 3000, 128)
    lay = cluster_layer(k, v, fp64_assign=False)
    q = torch.full((1, 8, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    cluster_topk_attention(q, lay, 5)
    w, lse = M.token_weights(q, lay)
    M.token_topk_attention(q, lay, 100, weights=w)
    M.adaptive_token_budget_batched(lay, w, 0.9)
    M.mixed_attention_f64(q, lay)
    lm = torch.zeros((1, 8, lay.cluster_cap), dtype=torch.float64, device="cuda")
    st = torch.zeros((1, 8, lay.cluster_cap), dtype=torch.uint8, device="cuda")
    cnt = torch.zeros((1, 8, 2), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    N.check(N.lib().dp_score(lay.view(), N.ptr(q), 1, 4, 1 / 128 ** 0.5, N.ptr(lm), s))
    N.check(N.lib().dp_select(lay.view(), 4, 0.95, 0.7, N.ptr(lm), N.ptr(st), N.ptr(cnt), None, None, None, None, 0,
                              s))
    torch.cuda.synchronize()
    q2 = torch.randn((1, 8, 128), device="cuda").to(torch.bfloat16)
    assert torch.isfinite(cluster_topk_attention(q2, lay, 5)).all()


@pytest.mark.parametrize("n,dtype", [(32768, torch.bfloat16), (8192, torch.float32), (131072, torch.bfloat16)])
def test_plan_split_equals_fused_plan(n, dtype):
    """dp_plan_score + dp_plan_given (config 5's split around an outside
    selection) fed the fused plan's OWN states reproduce the fused plan:
    identical log-masses and states, the same attention output."""
    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200 import cluster_layer
    from paper_2602_05191_b200.cache import dtype_code
    from paper_2602_05191_b200.workload import generate_layer, generate_queries

    H, G = (8, 4) if n <= 32768 else (2, 4)
    k, v, c = generate_layer(1, H, n, 128)
    lay = cluster_layer(k.to(dtype), v.to(dtype), fp64_assign=False)
    q = torch.from_numpy(generate_queries(c, G, 1)[0]).cuda().to(torch.bfloat16).contiguous()
    lib = N.lib()
    s = torch.cuda.current_stream().cuda_stream
    view = lay.view()
    cap = lay.cluster_cap
    wsb = lib.dp_decode_workspace_bytes(view, G)

    def run(split):
        lm = torch.full((1, H * G, cap), 7.0, dtype=torch.float64, device="cuda")
        st = torch.zeros((1, H * G, cap), dtype=torch.uint8, device="cuda")
        cnt = torch.zeros((1, H * G, 2), dtype=torch.int32, device="cuda")
        out = torch.zeros((1, H * G, 128), dtype=torch.float32, device="cuda")
        lse = torch.zeros((1, H * G), dtype=torch.float32, device="cuda")
        ws = torch.zeros((wsb,), dtype=torch.uint8, device="cuda")
        if split:
            N.check(lib.dp_plan_score(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(lm), N.ptr(ws), wsb, s))
            st.copy_(ref_state)
            N.check(lib.dp_plan_given(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(lm), N.ptr(st), 0, None,
                                      N.ptr(ws), wsb, s))
        else:
            N.check(lib.dp_plan(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, 0.95, 0.7, N.ptr(lm), N.ptr(st),
                                N.ptr(cnt), None, N.ptr(ws), wsb, s))
        N.check(lib.dp_attend(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(lm), N.ptr(out), N.ptr(lse),
                              N.ptr(ws), wsb, s))
        torch.cuda.synchronize()
        return lm, st, out, lse

    lm_a, st_a, out_a, lse_a = run(False)
    ref_state = st_a.clone()
    lm_b, st_b, out_b, lse_b = run(True)
    kk = lay.nclusters.reshape(-1).repeat_interleave(G)
    for r in range(H * G):
        K = int(kk[r])
        assert torch.equal(lm_a[0, r, :K], lm_b[0, r, :K]), r
        assert torch.all(lm_b[0, r, K:] == -math.inf), r  # score-only leaves -inf past K
    assert torch.equal(st_a, st_b)
    # the attention's cross-CTA accumulators are float atomics (order varies run to run)
    err = ((out_a - out_b).norm(dim=-1) / out_a.norm(dim=-1)).max().item()
    assert err <= 1e-6, err
    assert torch.allclose(lse_a, lse_b, rtol=0, atol=1e-5)
