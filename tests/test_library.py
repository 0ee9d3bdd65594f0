"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and validates arguments before touching the device."""

import ctypes

import numpy as np
import pytest

from paper_2602_05191_b200 import _native as N


def test_exports_every_header_symbol():
    lib = N.lib()
    syms = N.header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(N._SIGS) == set(syms)


def test_version_and_error_string():
    assert N.lib().dp_version() == 100
    assert isinstance(N.lib().dp_last_error(), bytes)


def _view(**kw):
    v = N.CacheView()
    v.batch, v.kv_heads, v.head_dim, v.dtype = 1, 8, 128, N.DP_BF16
    v.row_cap, v.n_tokens, v.sink, v.window, v.cluster_cap = 32768, 32768, 4, 64, 1022
    for k, val in kw.items():
        setattr(v, k, val)
    return v


def test_argument_validation_without_device():
    lib = N.lib()
    # p outside (0, 1] -> ValueError with the reference message
    with pytest.raises(ValueError, match="p1 must be in"):
        N.check(lib.dp_select(_view(), 4, 0.0, 0.7, None, None, None, None, None, None, None, 0, None))
    with pytest.raises(ValueError, match="p2 must be in"):
        N.check(lib.dp_select(_view(), 4, 0.9, 1.5, None, None, None, None, None, None, None, 0, None))
    with pytest.raises(ValueError, match="config/cache mismatch"):
        N.check(lib.dp_score(_view(sink=40000), None, 1, 4, 0.1, None, None))
    with pytest.raises(NotImplementedError):
        N.check(lib.dp_score(_view(head_dim=100), None, 1, 4, 0.1, None, None))
    with pytest.raises(NotImplementedError):
        N.check(lib.dp_score(_view(), None, 1, 16, 0.1, None, None))
    with pytest.raises(ValueError, match="workspace too small"):
        N.check(lib.dp_sparse_attention(_view(), None, 1, 4, 0.1, None, None, None, None, None, None, 0, None))
    p = N.ClusterParams()
    p.batch, p.kv_heads, p.head_dim, p.dtype = 1, 1, 64, 0
    p.n_tokens, p.sink, p.window, p.k, p.max_iters = 60, 4, 64, 1, 25
    with pytest.raises(ValueError, match="no middle tokens to cluster"):
        N.check(lib.dp_cluster_build(p, *([None] * 8), 0, None, None, None, None, 0, None, None, None, None, 0,
                                     None))
    p.n_tokens, p.k = 100, 50
    with pytest.raises(ValueError, match="more clusters than points"):
        N.check(lib.dp_kmeanspp(p, None, None, None, None, None, None, None, 0, None))


def test_workspace_sizes_are_host_computable():
    lib = N.lib()
    small = lib.dp_decode_workspace_bytes(_view(row_cap=8192, n_tokens=8192, cluster_cap=254), 4)
    big = lib.dp_decode_workspace_bytes(_view(), 4)
    assert 0 < small < big
    p = N.ClusterParams()
    p.batch, p.kv_heads, p.head_dim, p.dtype = 1, 8, 128, 1
    p.n_tokens, p.sink, p.window, p.k, p.max_iters = 32768, 4, 64, 1022, 25
    assert lib.dp_cluster_workspace_bytes(p) > 8 * 32700 * 8


def test_kernel_seam_validation_without_device():
    """dp_kn_* (the reference's kernels.py seam) reject bad arguments on the
    host, before any device work, with the reference's error classes."""
    from paper_2602_05191_b200 import kernels as K

    assert K.BACKEND == "b200"
    with pytest.raises(ValueError, match="zero-size"):
        K.logsumexp([])
    with pytest.raises(ValueError, match="zero-size"):
        K.softmax(np.zeros(0))
    with pytest.raises(IndexError):
        K.gather_scaled_logits(np.zeros((4, 2), np.float32), [4], np.zeros(2), 1.0)
    with pytest.raises(ValueError, match="empty sequence"):
        K.nearest_centroid(np.zeros((3, 2)), np.zeros((0, 2)))
    with pytest.raises(ValueError, match="not aligned"):
        K.weighted_sum(np.ones(3), np.ones((4, 2)))
    assert K.sorted_prefix_count([], 0.5) == 0
    assert K.scaled_logits(np.zeros((0, 3)), np.zeros(3), 1.0).shape == (0,)
    lib = N.lib()
    out = np.zeros(2)
    idx = np.array([0, 9], dtype=np.int64)
    with pytest.raises(ValueError, match="index out of range"):
        N.check(lib.dp_kn_scaled_logits(None, N.DP_F32, 4, 2, idx.ctypes.data, 2, None, 1.0, out.ctypes.data))
    with pytest.raises(ValueError, match="float32 or float64"):
        N.check(lib.dp_kn_scaled_logits(None, N.DP_BF16, 4, 2, None, 0, None, 1.0, out.ctypes.data))
