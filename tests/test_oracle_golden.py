"""Pin the CPU oracle against the real reference's outputs (tests/golden/,
made by oracle/gen_golden.py) and the reference's own known-answer tests
(SURVEY.md §8c).  CPU only."""

import glob
import hashlib
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import doublep_oracle as O

THRESHOLDS = [(0.95, 0.7), (0.99, 0.8), (0.9, 0.7), (1.0, 1.0), (0.5, 0.95)]
CASES = {
    "peaked_512_d16": dict(context_len=512, head_dim=16, num_kv_heads=2, gqa_group=2,
                           num_steps=2, tail_profile="peaked", seed=0),
    "mixed_1024_d32": dict(context_len=1024, head_dim=32, num_kv_heads=2, gqa_group=4,
                           num_steps=2, tail_profile="mixed", seed=3),
    "peaked_2048_d64": dict(context_len=2048, head_dim=64, num_kv_heads=1, gqa_group=4,
                            num_steps=2, tail_profile="peaked", seed=7),
    "heavy_1500_d128": dict(context_len=1500, head_dim=128, num_kv_heads=1, gqa_group=2,
                            num_steps=1, tail_profile="heavy", seed=11),
    "uniform_700_d16": dict(context_len=700, head_dim=16, num_kv_heads=1, gqa_group=2,
                            num_steps=1, tail_profile="uniform", seed=5),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_golden_fixtures_present():
    names = {os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))}
    assert set(CASES) <= names and "growth_300_d16" in names


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    spec = O.WorkloadSpec(**CASES[name])
    keys, values, queries = O.generate(spec)
    # generator is bit-identical to workload.generate
    assert sha(keys) == str(g["keys_sha"])
    assert sha(values) == str(g["values_sha"])
    assert sha(queries) == str(g["queries_sha"])
    tpc = int(g["tokens_per_cluster"])
    n, d = spec.context_len, spec.head_dim
    tables = {}
    for layer in range(spec.num_layers):
        for h in range(spec.num_kv_heads):
            pre = f"L{layer}H{h}_"
            k = O.clamp_k(n, spec.sink, spec.window, None, tpc)
            seed_h = O.head_seed(0, layer, h)
            mid = keys[layer, h, spec.sink:n - spec.window]
            centers, picks = O.plusplus_init(mid.astype(np.float64), k, np.random.default_rng(seed_h))
            np.testing.assert_array_equal(centers, g[pre + "init_centers"])
            # replayed stream reproduces the same picks (the device init path)
            first, u = O.init_stream(seed_h, mid.shape[0], k)
            assert first == picks[0] and u.shape == (k - 1,)
            t, fit = O.build_head_tables(keys[layer, h], values[layer, h], k, spec.sink,
                                         spec.window, seed_for_head=seed_h)
            np.testing.assert_array_equal(fit.assignments, g[pre + "assign"])
            np.testing.assert_allclose(fit.objective, g[pre + "objective"], rtol=1e-12)
            np.testing.assert_allclose(t.centroids, g[pre + "centroids"], rtol=0, atol=1e-12)
            np.testing.assert_allclose(t.value_means, g[pre + "value_means"], rtol=0, atol=1e-12)
            np.testing.assert_array_equal(t.sizes, g[pre + "sizes"])
            tables[layer, h] = t
    G = spec.gqa_group
    for ti, (p1, p2) in enumerate(THRESHOLDS):
        for s in range(spec.num_steps):
            for layer in range(spec.num_layers):
                for qh in range(spec.num_query_heads):
                    h = qh // G
                    pre = f"T{ti}S{s}L{layer}Q{qh}_"
                    q = queries[s, layer, qh]
                    out, pl, est = O.decode_step(q, keys[layer, h], values[layer, h],
                                                 tables[layer, h], p1, p2, spec.sink, spec.window)
                    np.testing.assert_allclose(est.log_masses, g[pre + "log_masses"], rtol=0, atol=1e-12)
                    np.testing.assert_array_equal(pl.stage1.selected, g[pre + "stage1"])
                    assert pl.stage1.cumulative_mass == pytest.approx(float(g[pre + "cum1"]), abs=1e-14)
                    assert pl.exact_clusters.size == int(g[pre + "n_exact"])
                    assert pl.exact_tokens.size == int(g[pre + "n_tokens"])
                    assert sha(pl.exact_tokens.astype(np.int64)) == str(g[pre + "tokens_sha"])
                    np.testing.assert_allclose(out.output, g[pre + "output"], rtol=1e-12, atol=1e-12)
                    assert out.normalizer == pytest.approx(float(g[pre + "normalizer"]), rel=1e-12)
                    if ti == 0:
                        full = O.full_attention(q, keys[layer, h], values[layer, h])
                        np.testing.assert_allclose(full.output, g[pre + "full_output"], rtol=1e-12, atol=1e-12)


def test_oracle_growth_matches_reference():
    g = np.load(os.path.join(GOLDEN, "growth_300_d16.npz"))
    spec = O.WorkloadSpec(context_len=300, head_dim=16, num_steps=1, tail_profile="peaked", seed=2)
    keys, values, queries = O.generate(spec)
    n = 300
    k = O.clamp_k(n, 4, 64)
    base, _ = O.build_head_tables(keys[0, 0], values[0, 0], k, 4, 64, seed_for_head=O.head_seed(0, 0, 0))
    kf = np.concatenate([keys[0, 0], g["app_k"][:, 0, 0]])
    vf = np.concatenate([values[0, 0], g["app_v"][:, 0, 0]])
    t = O.grow_tables(base, kf, vf, n, n + 5, 64)
    q = queries[0, 0, 0]
    for ti, (p1, p2) in enumerate([(1.0, 1.0), (0.9, 0.7)]):
        out, pl, _ = O.decode_step(q, kf, vf, t, p1, p2, 4, 64)
        np.testing.assert_array_equal(pl.stage1.selected, g[f"T{ti}_stage1"])
        np.testing.assert_array_equal(pl.exact_tokens, g[f"T{ti}_tokens"])
        np.testing.assert_allclose(out.output, g[f"T{ti}_output"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(O.full_attention(q, kf, vf).output, g["growth_full"], rtol=1e-10, atol=1e-12)


# --- the reference's own known-answer tests ---------

def test_kat_top_p():
    assert list(O.top_p_select([0.1, 0.6, 0.3], 0.95).selected) == [1, 2, 0]  # test_selection.py:29-31
    assert list(O.top_p_select([0.25, 0.5, 0.25], 0.75).selected) == [1, 0]  # :46-49
    assert sorted(O.top_p_select([0.6, 0.3, 0.1], 0.8).selected) == [0, 1]
    assert sorted(O.top_p_select([0.2, 0.5, 0.3], 1.0).selected) == [0, 1, 2]
    assert O.top_p_select_sorted([0.5, 0.5], 0.5) == 1
    assert O.top_p_select_sorted([0.6, 0.1, 0.9], 0.5) == 1
    with pytest.raises(ValueError):
        O.top_p_select_sorted([0.1, 0.6, 0.3], 0.5)


def test_kat_stage2_spec_example():
    # A=[0.5,0.3,0.2], p2=0.7 -> C_exact={0,1}
    cp = O.top_p_select(np.array([0.5, 0.3, 0.2]), 1.0).selected
    n2 = len(O.top_p_select(np.array([0.5, 0.3, 0.2])[cp], 0.7).selected)
    assert sorted(cp[:n2]) == [0, 1]


def test_kat_two_token_cluster():
    # test_engine.py:113-125: logits {0,2} in one cluster -> 2e vs 1+e^2
    keys = np.array([[0.0], [2.0]])
    t = O.HeadTables(members=[np.array([0, 1])], centroids=keys.mean(axis=0, keepdims=True),
                     value_means=np.ones((1, 1)))
    est = O.estimate(np.ones(1), t, 1)
    assert math.exp(est.log_masses[0]) == pytest.approx(2 * math.e, rel=1e-12)
    assert math.exp(est.log_masses[0]) == pytest.approx(5.4366, abs=1e-4)
    assert 1 + math.e ** 2 == pytest.approx(8.3891, abs=1e-4)


def test_kat_lse_and_tie():
    assert O.logsumexp([0.0, 2.0]) == pytest.approx(2.1269, abs=1e-4)  # test_numerics.py:21-26
    a, _ = O.nearest_centroid(np.zeros((1, 2)), np.array([[1.0, 0.0], [-1.0, 0.0]]))
    assert a[0] == 0  # test_kernels.py:79-84


def test_exhaustive_prefix_oracle_bulk():
    # test_selection.py:34-43 with the exhaustive prefix oracle
    rng = np.random.default_rng(42)
    for _ in range(300):
        n = int(rng.integers(1, 65))
        probs = rng.random(n)
        probs /= probs.sum()
        p = float(rng.uniform(0.05, 0.999))
        order = np.argsort(-probs, kind="stable")
        run, want = 0.0, order
        for i, idx in enumerate(order):
            run += probs[idx]
            if run / probs.sum() >= p:
                want = order[: i + 1]
                break
        assert np.array_equal(O.top_p_select(probs, p).selected, want)


def test_lse_merge_matches_whole():
    rng = np.random.default_rng(0)
    logits = rng.normal(size=100) * 4
    vals = rng.normal(size=(100, 8))
    lse = O.logsumexp(logits)
    whole = np.exp(logits - lse) @ vals
    parts = []
    for s in range(0, 100, 17):
        lg = logits[s:s + 17]
        m = lg.max()
        e = np.exp(lg - m)
        parts.append((m, e.sum(), e @ vals[s:s + 17] / e.sum()))
    parts.append((-np.inf, 0.0, np.zeros(8)))  # an empty shard
    M, L, o = O.lse_merge(*zip(*parts))
    np.testing.assert_allclose(o, whole, rtol=1e-12)
    assert M + math.log(L) == pytest.approx(lse, rel=1e-12)


def _seam():
    return np.load(os.path.join(GOLDEN, "kernels_seam.npz"))


def test_oracle_seam_matches_compiled_reference_backend():
    """The Cython-order restatements are bit-identical to the reference's
    compiled backend (_kernels_cy.pyx, tests/golden/kernels_seam.npz from
    oracle/gen_golden_seam.py); the reductions agree to the reference's own
    backend-parity tolerance (tests/test_kernels.py:30-67)."""
    g = _seam()
    for t in "abcde":
        keys, q, s = g[f"sl_{t}_keys"], g[f"sl_{t}_q"], float(g[f"sl_{t}_scale"])
        np.testing.assert_array_equal(O.scaled_logits_seq(keys, None, q, s), g[f"sl_{t}_out"])
        np.testing.assert_array_equal(O.scaled_logits_seq(keys, g[f"sl_{t}_idx"], q, s), g[f"sl_{t}_gout"])
        np.testing.assert_allclose(O.scaled_logits(keys, q, s), g[f"sl_{t}_out"], rtol=1e-12, atol=1e-12)
    for t in "abcd":
        x = g[f"lse_{t}_x"]
        assert O.logsumexp(x) == pytest.approx(float(g[f"lse_{t}_out"]), rel=1e-12, abs=1e-12)
        np.testing.assert_allclose(O.softmax(x), g[f"sm_{t}_out"], rtol=1e-12, atol=1e-15)
    assert O.logsumexp(g["lse_b_x"]) == float(g["lse_b_out"])  # exact for one element
    for t in "abc":
        w, mat, idx = g[f"ws_{t}_w"], g[f"ws_{t}_mat"], g[f"ws_{t}_idx"]
        np.testing.assert_allclose(O.weighted_sum(w, mat), g[f"ws_{t}_out"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(O.weighted_sum(w[: len(idx)], mat[idx]), g[f"ws_{t}_gout"], rtol=1e-12,
                                   atol=1e-12)
    for t in "abcde":
        a, b = O.nearest_centroid_direct(g[f"nc_{t}_pts"], g[f"nc_{t}_cents"])
        np.testing.assert_array_equal(a, g[f"nc_{t}_assign"])
        np.testing.assert_array_equal(b, g[f"nc_{t}_dsq"])
    assert g["nc_d_assign"][0] == 0 and not np.any(g["nc_e_assign"] == 5)  # ties -> lower index
    off = 0
    for n, p, c in zip(g["spc_lens"], g["spc_p"], g["spc_count"]):
        assert O.sorted_prefix_count(g["spc_vals"][off:off + n], p) == c
        off += n
    for p, c in zip(g["spc_big_p"], g["spc_big_count"]):
        assert O.sorted_prefix_count(g["spc_big"], p) == c
