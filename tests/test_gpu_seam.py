"""The reference's kernel plugin seam on the GPU (paper_2602_05191_b200.kernels
over dp_kn_*, csrc/seam.cu), checked like the reference checks its two
backends against each other (tests/test_kernels.py): against the compiled
reference backend's outputs (tests/golden/kernels_seam.npz, written by
_kernels_cy via oracle/gen_golden_seam.py) and the oracle.

Bar: scaled_logits, gather_scaled_logits, nearest_centroid and
sorted_prefix_count BIT-IDENTICAL to the Cython backend; logsumexp, softmax
and the weighted sums within the reference's rtol 1e-12."""

import os
import threading

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import doublep_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2602_05191_b200 import kernels

    return kernels


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "kernels_seam.npz"))


def test_backend_is_reported(K):
    assert K.BACKEND == "b200"


def test_scaled_logits_bit_identical(K, g):
    for t in "abcde":
        keys, q, s = g[f"sl_{t}_keys"], g[f"sl_{t}_q"], float(g[f"sl_{t}_scale"])
        np.testing.assert_array_equal(K.scaled_logits(keys, q, s), g[f"sl_{t}_out"])
        np.testing.assert_array_equal(K.gather_scaled_logits(keys, g[f"sl_{t}_idx"], q, s), g[f"sl_{t}_gout"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_scaled_logits_parity(K, dtype):
    rng = np.random.default_rng(0)
    keys = rng.normal(size=(4099, 96)).astype(dtype)
    q = rng.normal(size=96)
    np.testing.assert_array_equal(K.scaled_logits(keys, q, 0.25), O.scaled_logits_seq(keys, None, q, 0.25))
    idx = np.array([5, 0, 4098, 5, -1], dtype=np.intp)  # repeats and a negative index (NumPy wraps it)
    np.testing.assert_array_equal(K.gather_scaled_logits(keys, idx, q, 0.5),
                                  O.scaled_logits_seq(keys, idx, q, 0.5))
    with pytest.raises(IndexError):
        K.gather_scaled_logits(keys, [4099], q, 0.5)
    assert K.scaled_logits(keys[:0], q, 1.0).shape == (0,)
    # non-float inputs are coerced to float64 like the reference dispatcher
    ik = rng.integers(-3, 4, size=(17, 8))
    np.testing.assert_array_equal(K.scaled_logits(ik, np.ones(8), 1.0), ik.sum(axis=1).astype(np.float64))


def test_reductions(K, g):
    for t in "abcd":
        x = g[f"lse_{t}_x"]
        assert K.logsumexp(x) == pytest.approx(float(g[f"lse_{t}_out"]), rel=1e-12, abs=1e-12)
        np.testing.assert_allclose(K.softmax(x), g[f"sm_{t}_out"], rtol=1e-12, atol=1e-15)
    assert K.logsumexp(g["lse_b_x"]) == float(g["lse_b_out"])  # exact for a single element
    rng = np.random.default_rng(2)
    x = rng.normal(scale=30.0, size=300_001)  # multi-pass over one CTA
    assert K.logsumexp(x) == pytest.approx(O.logsumexp(x), rel=1e-12)
    np.testing.assert_allclose(K.softmax(x), O.softmax(x), rtol=1e-12, atol=1e-15)
    with pytest.raises(ValueError):
        K.logsumexp([])


def test_weighted_sums(K, g):
    for t in "abc":
        w, mat, idx = g[f"ws_{t}_w"], g[f"ws_{t}_mat"], g[f"ws_{t}_idx"]
        np.testing.assert_allclose(K.weighted_sum(w, mat), g[f"ws_{t}_out"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(K.gather_weighted_sum(w[: len(idx)], mat, idx), g[f"ws_{t}_gout"], rtol=1e-12,
                                   atol=1e-12)
    rng = np.random.default_rng(3)
    mat = rng.normal(size=(70_000, 40)).astype(np.float32)  # 274 partials
    w = rng.random(70_000)
    np.testing.assert_allclose(K.weighted_sum(w, mat), O.weighted_sum(w, mat), rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(K.weighted_sum(np.zeros(0), mat[:0]), np.zeros(40))
    with pytest.raises(ValueError):
        K.weighted_sum(w[:5], mat)


def test_nearest_centroid_bit_identical_and_ties(K, g):
    for t in "abcde":
        a, b = K.nearest_centroid(g[f"nc_{t}_pts"], g[f"nc_{t}_cents"])
        assert a.dtype == np.int64
        np.testing.assert_array_equal(a, g[f"nc_{t}_assign"])
        np.testing.assert_array_equal(b, g[f"nc_{t}_dsq"])
    # exact tie between two centroids: the lower index wins
    a, _ = K.nearest_centroid(np.zeros((1, 2)), np.array([[1.0, 0.0], [-1.0, 0.0]]))
    assert a[0] == 0
    # d large enough to shrink the per-CTA point tile
    rng = np.random.default_rng(4)
    pts, cents = rng.normal(size=(70, 700)), rng.normal(size=(6, 700))
    a, b = K.nearest_centroid(pts, cents)
    ea, eb = O.nearest_centroid_direct(pts, cents)
    np.testing.assert_array_equal(a, ea)
    np.testing.assert_array_equal(b, eb)


def test_sorted_prefix_count(K, g):
    off = 0
    for n, p, c in zip(g["spc_lens"], g["spc_p"], g["spc_count"]):
        assert K.sorted_prefix_count(g["spc_vals"][off:off + n], p) == c
        off += n
    for p, c in zip(g["spc_big_p"], g["spc_big_count"]):  # crosses the 4096-entry chunks
        assert K.sorted_prefix_count(g["spc_big"], p) == c
    with pytest.raises(ValueError, match="not sorted"):
        K.sorted_prefix_count(np.array([0.1, 0.6, 0.3]), 0.5)
    # an ascent past the stopping point is never scanned
    assert K.sorted_prefix_count(np.array([0.6, 0.3, 0.05, 0.9]), 0.5) == 1
    assert K.sorted_prefix_count(np.zeros(0), 0.5) == 0


def test_dispatcher_accepts_lists(K):
    assert K.logsumexp([0.0, 0.0]) == pytest.approx(np.log(2.0))
    np.testing.assert_allclose(K.softmax([1.0, 1.0]), [0.5, 0.5])


def test_threads_share_the_device(K):
    rng = np.random.default_rng(6)
    keys = rng.normal(size=(2000, 64)).astype(np.float32)
    qs = rng.normal(size=(8, 64))
    want = [O.scaled_logits_seq(keys, None, q, 0.125) for q in qs]
    got = [None] * 8

    def run(i):
        for _ in range(5):
            got[i] = K.scaled_logits(keys, qs[i], 0.125)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)
