"""GPU parity of the measurement side: true token
weights, the token top-k baseline, recovered mass, adaptive token budget and
cluster approximation error, all through the C ABI (metrics.cu), against the
reference's golden vectors (tests/golden/metrics_small.npz) and the CPU
oracle.  Everything is fp64 on both sides; selections are exact up to weight
ties within 1e-12 (relative), which the tests classify instead of passing."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import doublep_oracle as O
from parity import oracle_tables

pytestmark = pytest.mark.gpu

TOKEN_BUDGETS = [1, 17, 200]
PS = [0.5, 0.9, 0.95, 0.99]
PLANS = [(0.95, 0.7), (0.9, 0.7)]
WTIE = 1e-12


def _same_set_modulo_ties(w, got, want):
    """Equal-size index sets hold the same weights up to ties within WTIE."""
    a = np.sort(w[sorted(got - want)]) if got - want else np.empty(0)
    b = np.sort(w[sorted(want - got)]) if want - got else np.empty(0)
    scale = max(float(w.max()), 1e-300)
    return a.size == b.size and bool(np.all(np.abs(a - b) <= WTIE * scale))


def _budget_ok(w, got, want, p):
    """Adaptive budgets agree, or differ only where the sorted cumulative
    mass sits within 1e-9 of p (fp64 summation order)."""
    if got == want:
        return True
    cum = np.cumsum(np.sort(w)[::-1])
    lo, hi = sorted((got, want))
    return all(abs(cum[j - 1] - p) <= 1e-9 for j in range(lo, min(hi, cum.size) + 1))


@pytest.mark.parametrize("tag", ["A_", "T_"])
def test_reference_signatures_match_golden(tag):
    """Reference-signature wrappers (KvCache in, numpy out) against the real
    reference's values, including the duplicated-row cache whose weights tie
    in pairs (lower position must win)."""
    from paper_2602_05191_b200 import KvCache, build_clustered_cache, metrics as M
    from paper_2602_05191_b200 import DoublePConfig, decode_step

    g = np.load(os.path.join(GOLDEN, "metrics_small.npz"))
    keys, values, queries = g[tag + "keys"], g[tag + "values"], g[tag + "queries"]
    sink, window = (int(x) for x in g[tag + "sink_window"])
    S, L, Hq, d = queries.shape
    H, n = keys.shape[1], keys.shape[2]
    G = Hq // H
    cache = KvCache(torch.from_numpy(keys), torch.from_numpy(values))
    cc = build_clustered_cache(cache, sink=sink, window=window)
    for s in range(S):
        for layer in range(L):
            for qh in range(Hq):
                h = qh // G
                q = torch.from_numpy(queries[s, layer, qh].copy())
                pre = f"{tag}S{s}L{layer}Q{qh}_"
                w, lse = M.full_attention_weights(q, cache, layer, h)
                wo, lo = O.full_attention_weights(queries[s, layer, qh].astype(np.float64), keys[layer, h])
                np.testing.assert_allclose(w, wo, rtol=1e-12, atol=1e-300)
                assert lse == pytest.approx(lo, rel=1e-13, abs=1e-13)
                for bud in TOKEN_BUDGETS + [n]:
                    out, cap = M.baseline_token_topk(q, cache, bud, layer, h)
                    np.testing.assert_allclose(out.output, g[pre + f"tk{bud}_out"], rtol=1e-11, atol=1e-12)
                    assert cap == pytest.approx(float(g[pre + f"tk{bud}_cap"]), rel=1e-11)
                    assert out.normalizer == pytest.approx(float(g[pre + f"tk{bud}_norm"]), rel=1e-11)
                for i, p in enumerate(PS):
                    got = M.adaptive_token_budget(q, cache, p, layer, h)
                    assert _budget_ok(wo, got, int(g[pre + f"ab{i}"]), p), (pre, p, got)
                for i, (p1, p2) in enumerate(PLANS):
                    cfg = DoublePConfig(p1=p1, p2=p2, sink=sink, window=window)
                    _, plan, _ = decode_step(q, cache, cc, cfg, layer, h)
                    # the GPU plan's exact tokens, re-measured by the oracle on the true weights
                    want = O.recovered_mass(wo, plan.exact_tokens)
                    assert M.recovered_mass(plan, q, cache) == pytest.approx(want, rel=1e-12)
                err, order = M.cluster_approx_error(q, cache, cc, layer, h)
                t = oracle_tables(cc.layers[layer], 0, h)
                est = O.estimate(queries[s, layer, qh].astype(np.float64), t, d)
                # estimate from the GPU tables (fp32 centroids): same order up to ties
                e_o, ord_o = O.cluster_approx_error(wo, lo, est, t)
                if np.array_equal(order, ord_o):
                    np.testing.assert_allclose(err, e_o, rtol=1e-9, atol=1e-14)
    with pytest.raises(ValueError, match="budget must be in"):
        M.baseline_token_topk(torch.from_numpy(queries[0, 0, 0].copy()), cache, n + 1, 0, 0)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_batched_metrics_parity(dtype):
    """Batched device API over a clustered layer (B=2, G=4): weights, token
    top-k sets/outputs, recovered mass of the fused plan, adaptive budgets and
    cluster errors against the oracle fed the GPU's own tables."""
    from paper_2602_05191_b200 import cluster_layer, sparse_attention
    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200 import metrics as M

    B, H, G, n, d = 2, 2, 4, 3000, 128
    ks, vs, qs = [], [], []
    for b in range(B):
        spec = O.WorkloadSpec(context_len=n, head_dim=d, num_kv_heads=H, gqa_group=G, num_steps=1,
                              tail_profile="mixed", seed=40 + b)
        keys, values, queries = O.generate(spec)
        ks.append(keys[0])
        vs.append(values[0])
        qs.append(queries[0, 0])
    kd = torch.from_numpy(np.stack(ks)).cuda().to(dtype)
    vd = torch.from_numpy(np.stack(vs)).cuda().to(dtype)
    q = torch.from_numpy(np.stack(qs)).cuda().to(dtype)
    layer = cluster_layer(kd, vd, fp64_assign=False)
    out_sp, ws = sparse_attention(q, layer, 0.95, 0.7, return_plan=True)
    w, lse = M.token_weights(q, layer)
    budget = 333
    tk_out, tk_cap, sel = M.token_topk_attention(q, layer, budget, weights=w, return_selected=True)
    rec = M.recovered_mass_batched(layer, w, ws.state)
    ab = M.adaptive_token_budget_batched(layer, w, 0.9)
    order = torch.zeros_like(ws.state, dtype=torch.int32)
    st2, c2 = torch.zeros_like(ws.state), torch.zeros_like(ws.counts)
    N.check(N.lib().dp_select(layer.view(), G, 1.0, 1.0, N.ptr(ws.log_mass), N.ptr(st2), N.ptr(c2), N.ptr(order),
                              None, None, None, 0, torch.cuda.current_stream().cuda_stream))
    cae = M.cluster_approx_error_batched(layer, w, lse, ws.log_mass, order)
    torch.cuda.synchronize()
    kf = kd.double().cpu().numpy()
    vf = vd.double().cpu().numpy()
    for b in range(B):
        for hq in range(H * G):
            h = hq // G
            qv = q[b, hq].double().cpu().numpy()
            wo, lo = O.full_attention_weights(qv, kf[b, h])
            wg = M.to_positions(layer, w[b, hq], b, h)
            np.testing.assert_allclose(wg, wo, rtol=1e-12, atol=1e-300)
            assert float(lse[b, hq]) == pytest.approx(lo, rel=1e-13, abs=1e-13)
            # token top-k: same set (modulo ties), same output
            sel_pos = set(np.flatnonzero(M.to_positions(layer, sel[b, hq], b, h)).tolist())
            o_out, o_cap, o_idx = O.token_topk(qv, kf[b, h], vf[b, h], budget)
            assert len(sel_pos) == budget
            assert _same_set_modulo_ties(wo, sel_pos, set(o_idx.tolist())), (b, hq)
            if sel_pos == set(o_idx.tolist()):
                np.testing.assert_allclose(tk_out[b, hq].cpu().numpy(), o_out.output, rtol=1e-11, atol=1e-12)
                assert float(tk_cap[b, hq]) == pytest.approx(o_cap, rel=1e-11)
            # recovered mass of the fused plan's exact set
            t = oracle_tables(layer, b, h)
            st = ws.state[b, hq].cpu().numpy()
            K = len(t.members)
            exact = np.concatenate([np.arange(layer.sink), np.arange(n - layer.window, n),
                                    *[t.members[c] for c in range(K) if st[c] == 2]])
            assert float(rec[b, hq]) == pytest.approx(O.recovered_mass(wo, exact), rel=1e-12)
            assert _budget_ok(wo, int(ab[b, hq]), O.adaptive_token_budget(wo, 0.9), 0.9)
            est = O.estimate(qv, t, d)
            e_o, ord_o = O.cluster_approx_error(wo, lo, est, t)
            og = order[b, hq, :K].cpu().numpy()
            if np.array_equal(og, ord_o):
                np.testing.assert_allclose(cae[b, hq, :K].cpu().numpy(), e_o, rtol=1e-9, atol=1e-14)


def test_token_topk_ties_lower_position():
    """Duplicated key rows give pairwise-equal weights; an odd budget splits
    a pair, and the lower token position must be kept (selection.py:85-92)."""
    from paper_2602_05191_b200 import metrics as M
    from paper_2602_05191_b200.cache import ClusteredLayer

    rng = np.random.default_rng(5)
    n, d = 1000, 64
    base = rng.normal(size=(n // 2, d)).astype(np.float32)
    k = torch.from_numpy(np.repeat(base, 2, axis=0)).cuda().view(1, 1, n, d)
    v = torch.from_numpy(rng.normal(size=(n, d)).astype(np.float32)).cuda().view(1, 1, n, d)
    di = torch.zeros((1, 1, 2), dtype=torch.int32, device="cuda")
    df = torch.zeros((1, 1, 1, d), dtype=torch.float32, device="cuda")
    lay = ClusteredLayer(k, v, di, di[..., 0], df, df, None, n, 0, 0)
    q = torch.from_numpy(rng.normal(size=(1, 1, d)).astype(np.float32) * 3).cuda()
    for budget in (1, 7, 99, 501, n):
        out, cap, sel = M.token_topk_attention(q, lay, budget, return_selected=True)
        got = np.flatnonzero(sel[0, 0, :n].cpu().numpy())
        o_out, o_cap, idx = O.token_topk(q[0, 0].double().cpu().numpy(), k[0, 0].double().cpu().numpy(),
                                         v[0, 0].double().cpu().numpy(), budget)
        np.testing.assert_array_equal(got, np.sort(idx))
        np.testing.assert_allclose(out[0, 0].cpu().numpy(), o_out.output, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_mixed_attention_f64_matches_oracle(dtype):
    """dp_mixed_attention_f64 (the runner's fp64 evaluation path) on the fused
    plan's states equals the oracle's mixed_attention fed the same GPU tables
    to fp64 rounding (1e-12), and with no states equals full attention."""
    from paper_2602_05191_b200 import cluster_layer, sparse_attention
    from paper_2602_05191_b200 import metrics as M

    B, H, G, n, d = 1, 2, 4, 2500, 64
    spec = O.WorkloadSpec(context_len=n, head_dim=d, num_kv_heads=H, gqa_group=G, num_steps=1,
                          tail_profile="mixed", seed=77)
    keys, values, queries = O.generate(spec)
    kd = torch.from_numpy(keys[0]).cuda().to(dtype).unsqueeze(0)
    vd = torch.from_numpy(values[0]).cuda().to(dtype).unsqueeze(0)
    q = torch.from_numpy(queries[0, 0]).cuda().to(dtype).unsqueeze(0)
    layer = cluster_layer(kd, vd, fp64_assign=False)
    _, ws = sparse_attention(q, layer, 0.9, 0.7, return_plan=True)
    out, lse = M.mixed_attention_f64(q, layer, ws.state, ws.log_mass)
    full, flse = M.mixed_attention_f64(q, layer)
    kf, vf = kd[0].double().cpu().numpy(), vd[0].double().cpu().numpy()
    st = ws.state[0].cpu().numpy()
    lm = ws.log_mass[0].cpu().numpy()
    for hq in range(H * G):
        h = hq // G
        t = oracle_tables(layer, 0, h)
        K = len(t.members)
        qv = q[0, hq].double().cpu().numpy()
        exact = np.sort(np.concatenate([np.arange(layer.sink), np.arange(n - layer.window, n),
                                        *[t.members[c] for c in range(K) if st[hq, c] == 2]]))
        approx = np.array([c for c in range(K) if st[hq, c] == 1], dtype=np.int64)
        est = O.Estimate(log_masses=lm[hq, :K], probs=None, order=None)
        ref = O.mixed_attention(qv, kf[h], vf[h], t, exact, approx, est)
        assert O.output_error(out[0, hq].cpu().numpy(), ref.output) <= 1e-12
        assert float(lse[0, hq]) == pytest.approx(ref.log_normalizer, abs=1e-12)
        dense = O.full_attention(qv, kf[h], vf[h])
        assert O.output_error(full[0, hq].cpu().numpy(), dense.output) <= 1e-12
