"""CPU tests of the host-side logic of the package (no device needed)."""

import numpy as np
import pytest

from oracle import doublep_oracle as O


def test_rng_stream_replays_plusplus_draws():
    """The host stream (first pick + uniforms) the device k-means++ consumes
    equals the draws `_plusplus_init` makes (clustering.py:41-52)."""
    from paper_2602_05191_b200.cache import head_seed, rng_stream

    rng = np.random.default_rng(123)
    f = int(rng.integers(1000))
    u = [rng.random() for _ in range(99)]
    f2, u2, _ = rng_stream(123, 1000, 100)
    assert f == f2 and np.array_equal(np.array(u), u2)
    # degenerate tail: rng.integers from the first zero-mass step on
    rng = np.random.default_rng(5)
    f = int(rng.integers(50))
    uu = [rng.random() for _ in range(9)]
    aa = [int(rng.integers(50)) for _ in range(10)]
    f3, u3, a3 = rng_stream(5, 50, 20, degenerate_from=10)
    assert f3 == f and np.array_equal(u3[:9], uu) and list(a3[9:]) == aa
    assert head_seed(0, 3, 5) == O.head_seed(0, 3, 5)


def test_replayed_stream_reproduces_reference_picks():
    """searchsorted(cumsum(dsq/total)/cdf[-1], u, 'right') with the replayed
    uniforms picks exactly what plusplus_init (pinned to the reference) picks."""
    from paper_2602_05191_b200.cache import rng_stream

    rng = np.random.default_rng(0)
    x = rng.normal(size=(500, 16))
    k = 40
    _, want = O.plusplus_init(x, k, np.random.default_rng(77))
    first, u, _ = rng_stream(77, 500, k)
    picks = [first]
    dsq = np.sum((x - x[first]) ** 2, axis=1)
    for i in range(1, k):
        p = dsq / dsq.sum()
        cdf = p.cumsum()
        cdf /= cdf[-1]
        idx = int(cdf.searchsorted(u[i - 1], side="right"))
        picks.append(idx)
        np.minimum(dsq, np.sum((x - x[idx]) ** 2, axis=1), out=dsq)
    np.testing.assert_array_equal(picks, want)


def test_config_validation_matches_reference():
    from paper_2602_05191_b200 import PRESETS, DoublePConfig

    with pytest.raises(ValueError):
        DoublePConfig(p1=0.0, p2=0.5)
    with pytest.raises(ValueError):
        DoublePConfig(p1=0.5, p2=1.0001)
    with pytest.raises(ValueError):
        DoublePConfig(p1=0.5, p2=0.5, sink=-1)
    assert PRESETS == {"llama-default": (0.95, 0.7), "qwen-default": (0.99, 0.8)}
    assert DoublePConfig(0.9, 0.7).cluster_count_for(8124) == 254


def test_cluster_geometry_errors():
    from paper_2602_05191_b200.cache import _check_geometry, default_cluster_count

    assert default_cluster_count(32700) == 1022
    assert _check_geometry(8192, 4, 64, None, 32) == (254, 8124)
    assert _check_geometry(100, 4, 64, 500, 32) == (32, 32)  # clamp to middle
    with pytest.raises(ValueError, match="no middle tokens to cluster"):
        _check_geometry(68, 4, 64, None, 32)
    with pytest.raises(ValueError, match="cluster count must be >= 1"):
        _check_geometry(100, 4, 64, 0, 32)


def test_query_law_matches_reference_directions():
    """The device workload's query law (multi-blob direction) equals the
    oracle's restatement of workload.py:104-127."""
    from paper_2602_05191_b200.workload import _multi_blob_direction

    rng = np.random.default_rng(1)
    centers = rng.normal(size=(8, 32))
    for chosen in ([0, 3], [1, 2, 5], [7, 4]):
        np.testing.assert_allclose(_multi_blob_direction(centers, chosen),
                                   O._multi_blob_direction(centers, chosen), rtol=1e-12)
