"""Pin the oracle's measurement-side functions (token top-k baseline, cluster
top-k baseline, recovered mass, adaptive budget, cluster approximation
error) against the real reference's outputs in tests/golden/metrics_small.npz
(made by oracle/gen_golden_metrics.py).  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import doublep_oracle as O

TOKEN_BUDGETS = [1, 17, 200]
CLUSTER_BUDGETS = [1, 3, 9]
PS = [0.5, 0.9, 0.95, 0.99]
PLANS = [(0.95, 0.7), (0.9, 0.7)]


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "metrics_small.npz"))


@pytest.mark.parametrize("tag", ["A_", "T_"])
def test_oracle_metrics_match_reference(golden, tag):
    g = golden
    keys, values, queries = g[tag + "keys"], g[tag + "values"], g[tag + "queries"]
    sink, window = (int(x) for x in g[tag + "sink_window"])
    S, L, Hq, d = queries.shape
    H = keys.shape[1]
    G = Hq // H
    n = keys.shape[2]
    tables = {}
    for layer in range(L):
        for h in range(H):
            k = O.clamp_k(n, sink, window)
            tables[layer, h], _ = O.build_head_tables(keys[layer, h], values[layer, h], k, sink, window,
                                                      seed_for_head=O.head_seed(0, layer, h))
    ties_seen = 0
    for s in range(S):
        for layer in range(L):
            for qh in range(Hq):
                h = qh // G
                q = queries[s, layer, qh].astype(np.float64)
                kh, vh, t = keys[layer, h], values[layer, h], tables[layer, h]
                pre = f"{tag}S{s}L{layer}Q{qh}_"
                w, lse = O.full_attention_weights(q, kh)
                for bud in TOKEN_BUDGETS + [n]:
                    out, cap, idx = O.token_topk(q, kh, vh, bud)
                    np.testing.assert_array_equal(np.sort(idx), g[pre + f"tk{bud}_set"])
                    np.testing.assert_allclose(out.output, g[pre + f"tk{bud}_out"], rtol=1e-12, atol=1e-12)
                    assert cap == pytest.approx(float(g[pre + f"tk{bud}_cap"]), rel=1e-12)
                    assert out.normalizer == pytest.approx(float(g[pre + f"tk{bud}_norm"]), rel=1e-12)
                    kth = np.sort(w)[::-1][bud - 1]
                    ties_seen += int(np.sum(w == kth) > 1)
                for bud in CLUSTER_BUDGETS:
                    out = O.cluster_topk(q, kh, vh, t, bud, sink, window)
                    np.testing.assert_allclose(out.output, g[pre + f"ck{bud}_out"], rtol=1e-12, atol=1e-12)
                for i, p in enumerate(PS):
                    assert O.adaptive_token_budget(w, p) == int(g[pre + f"ab{i}"])
                for i, (p1, p2) in enumerate(PLANS):
                    _, pl, _ = O.decode_step(q, kh, vh, t, p1, p2, sink, window)
                    assert O.recovered_mass(w, pl.exact_tokens) == pytest.approx(float(g[pre + f"rm{i}"]),
                                                                                 rel=1e-12)
                est = O.estimate(q, t, d)
                err, order = O.cluster_approx_error(w, lse, est, t)
                np.testing.assert_array_equal(order, g[pre + "cae_order"])
                np.testing.assert_allclose(err, g[pre + "cae_err"], rtol=1e-10, atol=1e-15)
    if tag == "T_":
        assert ties_seen > 0  # the duplicated-row cache really exercises the tie rule


def test_violation_rate():
    assert O.violation_rate([0.9, 0.96, 0.5, 0.99], 0.95) == 0.5
    with pytest.raises(ValueError):
        O.violation_rate([], 0.9)
