"""The reference's kernel plugin seam on the GPU: a ``DOUBLEP_KERNELS``
backend module.

The reference dispatches its eight per-query hot loops through
``doublep/kernels.py:47-96`` to ``_kernels_cy`` or ``_kernels_py``; this
module has the same names, argument meaning, coercions and error classes and
runs each one through libdoublep_b200.so's host-pointer entry points
(``dp_kn_*``, include/doublep_b200.h, csrc/seam.cu).  A maintainer adds it as
a third backend choice; ``integration.install_kernels`` does
that binding for a loaded ``doublep``.

Numerics (the reference's backend-parity contract, tests/test_kernels.py):
``scaled_logits``, ``gather_scaled_logits``, ``nearest_centroid`` and
``sorted_prefix_count`` are bit-identical to the Cython backend;
``logsumexp``, ``softmax`` and the weighted sums are tree-ordered fp64
reductions within 1e-12 relative.  No CPU fallback: without the library (or a
GPU) these raise.
"""

import ctypes

import numpy as np

from . import _native

BACKEND = "b200"


def _as_f64_vec(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _as_mat(x):
    """Reference coercion (kernels.py:35-39): float32/float64 kept, else f64."""
    a = np.ascontiguousarray(x)
    if a.dtype != np.float32 and a.dtype != np.float64:
        a = a.astype(np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {a.shape}")
    return a


def _as_idx(idx, rows):
    """kernels.py:42-43 (intp), with NumPy's indexing rules: negative indices
    wrap, out-of-range ones raise IndexError."""
    i = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1)
    if i.size and (i.min() < -rows or i.max() >= rows):
        bad = int(i[(i < -rows) | (i >= rows)][0])
        raise IndexError(f"index {bad} is out of bounds for axis 0 with size {rows}")
    return np.where(i < 0, i + rows, i).astype(np.int64) if i.size and i.min() < 0 else i


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _dtype(a):
    return _native.DP_F32 if a.dtype == np.float32 else _native.DP_F64


def _call(name, *args):
    _native.check(getattr(_native.lib(), name)(*args))


def _logits(keys, idx, q, scale):
    n = keys.shape[0] if idx is None else idx.shape[0]
    if q.shape[0] != keys.shape[1]:
        raise ValueError(f"shapes {keys.shape} and {q.shape} not aligned")
    out = np.empty(n, dtype=np.float64)
    _call("dp_kn_scaled_logits", _p(keys), _dtype(keys), keys.shape[0], keys.shape[1],
          None if idx is None else _p(idx), 0 if idx is None else idx.shape[0], _p(q), float(scale), _p(out))
    return out


def scaled_logits(keys, q, scale):
    """(keys @ q) * scale with float64 accumulation; float64[n]
    (kernels.py:47-49)."""
    return _logits(_as_mat(keys), None, _as_f64_vec(q), scale)


def gather_scaled_logits(keys, idx, q, scale):
    """scaled_logits over the rows of ``keys`` listed in ``idx``
    (kernels.py:52-56)."""
    keys = _as_mat(keys)
    return _logits(keys, _as_idx(idx, keys.shape[0]), _as_f64_vec(q), scale)


def logsumexp(x):
    """Max-subtracted log(sum(exp(x))) of a nonempty vector (kernels.py:59-61)."""
    x = _as_f64_vec(x).reshape(-1)
    out = np.empty(1, dtype=np.float64)
    _call("dp_kn_logsumexp", _p(x), x.shape[0], _p(out))
    return float(out[0])


def softmax(x):
    """Max-subtracted softmax of a nonempty vector; float64 (kernels.py:64-66)."""
    x = _as_f64_vec(x).reshape(-1)
    out = np.empty(x.shape[0], dtype=np.float64)
    _call("dp_kn_softmax", _p(x), x.shape[0], _p(out))
    return out


def _wsum(w, mat, idx):
    n = mat.shape[0] if idx is None else idx.shape[0]
    if w.shape[0] != n:
        raise ValueError(f"shapes ({w.shape[0]},) and ({n},{mat.shape[1]}) not aligned")
    out = np.zeros(mat.shape[1], dtype=np.float64)
    _call("dp_kn_weighted_sum", _p(w), _p(mat), _dtype(mat), mat.shape[0], mat.shape[1],
          None if idx is None else _p(idx), 0 if idx is None else idx.shape[0], _p(out))
    return out


def weighted_sum(weights, mat):
    """weights @ mat with float64 accumulation; float64[d] (kernels.py:69-71)."""
    return _wsum(_as_f64_vec(weights).reshape(-1), _as_mat(mat), None)


def gather_weighted_sum(weights, mat, idx):
    """weights @ mat[idx] with float64 accumulation (kernels.py:74-76)."""
    mat = _as_mat(mat)
    return _wsum(_as_f64_vec(weights).reshape(-1), mat, _as_idx(idx, mat.shape[0]))


def nearest_centroid(points, centroids):
    """Per-point closest centroid under squared Euclidean distance; (int64[n]
    assignments, float64[n] squared distances), ties to the lowest index
    (kernels.py:79-87)."""
    pts = _as_mat(points)
    cents = np.ascontiguousarray(centroids, dtype=np.float64)
    if cents.ndim != 2 or cents.shape[1] != pts.shape[1]:
        raise ValueError(f"centroids shape {cents.shape} does not match points {pts.shape}")
    n = pts.shape[0]
    assign = np.empty(n, dtype=np.int64)
    best = np.empty(n, dtype=np.float64)
    _call("dp_kn_nearest_centroid", _p(pts), _dtype(pts), n, pts.shape[1], _p(cents), cents.shape[0],
          _p(assign), _p(best))
    return assign, best


def sorted_prefix_count(sorted_probs, p):
    """Smallest prefix of a non-increasing vector with cumulative sum >= p;
    ValueError("input not sorted") on an ascent among the scanned entries
    (kernels.py:90-96)."""
    x = _as_f64_vec(sorted_probs).reshape(-1)
    out = np.zeros(1, dtype=np.int64)
    _call("dp_kn_sorted_prefix_count", _p(x), x.shape[0], float(p), _p(out))
    return int(out[0])
