"""ctypes binding of libdoublep_b200.so (C ABI in include/doublep_b200.h).

The product path has no CPU fallback: if the library is missing or fails to
load, importing the ops raises.  Status codes map to the reference's error
classes (DP_ERR_INVALID -> ValueError with the reference message).
"""

import ctypes
import os
import re

from .build import INCLUDE, LIB

DP_OK, DP_ERR_INVALID, DP_ERR_CUDA, DP_ERR_UNSUPPORTED = 0, 1, 2, 3
DP_F32, DP_BF16, DP_F64 = 0, 1, 2

_c_int_p = ctypes.POINTER(ctypes.c_int32)
_c_dbl_p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class CacheView(ctypes.Structure):
    """Mirror of dp_cache_view."""

    _fields_ = [
        ("batch", ctypes.c_int32), ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("row_cap", ctypes.c_int32), ("n_tokens", ctypes.c_int32),
        ("sink", ctypes.c_int32), ("window", ctypes.c_int32), ("cluster_cap", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("keys", _vp), ("values", _vp), ("offs", _vp), ("nclusters", _vp),
        ("centroids", _vp), ("value_means", _vp),
    ]


class ClusterParams(ctypes.Structure):
    """Mirror of dp_cluster_params."""

    _fields_ = [
        ("batch", ctypes.c_int32), ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("n_tokens", ctypes.c_int32), ("sink", ctypes.c_int32),
        ("window", ctypes.c_int32), ("k", ctypes.c_int32), ("max_iters", ctypes.c_int32),
        ("fp64_assign", ctypes.c_int32),
    ]


_SIGS = {
    "dp_version": (ctypes.c_int, []),
    "dp_last_error": (ctypes.c_char_p, []),
    "dp_device_info": (ctypes.c_int, [_c_int_p, _c_int_p, _c_int_p]),
    "dp_decode_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(CacheView), ctypes.c_int32]),
    "dp_score": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_double, _vp, _vp]),
    "dp_select": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int32, ctypes.c_double,
                                 ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t,
                                 _vp]),
    "dp_sparse_attention": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_double, _vp, _vp, _vp, _vp, _vp,
                                           _vp, ctypes.c_size_t, _vp]),
    "dp_build_worklist": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int32, _vp, _vp, _vp, _vp,
                                         ctypes.c_size_t, _vp]),
    "dp_attend": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_double, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_plan": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_plan_score": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                     _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_plan_given": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                     _vp, _vp, ctypes.c_int32, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_debug_plan_timing": (ctypes.c_int, [_vp]),
    "dp_debug_plan_clock": (ctypes.c_int, [_vp]),
    "dp_debug_attn_timing": (ctypes.c_int, [_vp]),
    "dp_debug_set": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "dp_debug_step_timing": (ctypes.c_int, [_vp]),
    "dp_debug_step_cluster_size": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int]),
    "dp_debug_plan_occupancy": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int, ctypes.c_int]),
    "dp_decode_step": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp, _vp,
                                      _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_cluster_topk": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_double, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_size_t, _vp]),
    "dp_dense_attention": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_double, _vp, _vp, _vp,
                                          ctypes.c_size_t, _vp]),
    "dp_token_weights": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_double, _vp, _vp, _vp]),
    "dp_token_topk": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     _vp, _vp, _vp, _vp, _vp, _vp]),
    "dp_recovered_mass": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int32, _vp, _vp, _vp, _vp]),
    "dp_cluster_approx_error": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int32, _vp, _vp, _vp, _vp, _vp,
                                               _vp]),
    "dp_adaptive_token_budget": (ctypes.c_int, [ctypes.POINTER(CacheView), ctypes.c_int32, _vp, ctypes.c_double,
                                                _vp, _vp]),
    "dp_mixed_attention_f64": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_double, _vp, _vp, _vp, _vp, _vp]),
    "dp_append_token": (ctypes.c_int, [ctypes.POINTER(CacheView), _vp, _vp, _vp]),
    "dp_cluster_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(ClusterParams)]),
    "dp_cluster_build": (ctypes.c_int, [ctypes.POINTER(ClusterParams), _vp, _vp, _vp, _vp, _vp, _vp,
                                        _vp, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp,
                                        ctypes.c_int32, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_kmeanspp": (ctypes.c_int, [ctypes.POINTER(ClusterParams), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   ctypes.c_size_t, _vp]),
    "dp_nearest_centroid": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp,
                                           ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp]),
    "dp_kmpp_shard_dsq": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp,
                                         ctypes.c_int32, _vp, _vp, _vp]),
    "dp_kmpp_shard_pick": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp,
                                          _vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.c_int64, _vp, _vp,
                                          _vp]),
    "dp_lloyd_shard_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "dp_lloyd_shard_sums": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp,
                                           ctypes.c_int32, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_select_global_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "dp_select_global": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_double, ctypes.c_double,
                                        _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_select_global_parts": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp,
                                              ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dp_lse_merge": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp]),
    "dp_kn_scaled_logits": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int64,
                                           _vp, ctypes.c_double, _vp]),
    "dp_kn_logsumexp": (ctypes.c_int, [_vp, ctypes.c_int64, _vp]),
    "dp_kn_softmax": (ctypes.c_int, [_vp, ctypes.c_int64, _vp]),
    "dp_kn_weighted_sum": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, _vp,
                                          ctypes.c_int64, _vp]),
    "dp_kn_nearest_centroid": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int32,
                                              _vp, _vp]),
    "dp_kn_sorted_prefix_count": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_double, _vp]),
}

_lib = None


def header_symbols():
    """Every dp_* entry point declared in include/doublep_b200.h."""
    with open(os.path.join(INCLUDE, "doublep_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(dp_[a-z_0-9]+)\s*\(", text)))


def lib():
    """Load (building first if absent) the shared library.  Raises if it
    cannot be loaded -- there is deliberately no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    from .build import build

    try:
        build()  # no-op when the library matches the sources' digest; rebuilds a stale one
    except FileNotFoundError:  # no nvcc on this host: use the prebuilt library if there is one
        if not os.path.exists(LIB):
            raise
        import warnings

        warnings.warn("nvcc not found: loading the prebuilt libdoublep_b200.so without a digest check")
    handle = ctypes.CDLL(LIB)
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


class DoublePError(RuntimeError):
    pass


def check(rc):
    if rc == DP_OK:
        return
    msg = lib().dp_last_error().decode()
    if rc == DP_ERR_INVALID:
        raise ValueError(msg)
    if rc == DP_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise DoublePError(msg)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())
