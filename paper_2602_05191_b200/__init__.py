"""B200-native Double-P hierarchical top-p sparse decode attention.

Drop-in for the decode path of the reference package ``doublep``
(arxiv 2602.05191): clustered KV-cache build at prefill, then a per-step
``sparse_attention(q, cache, p)``.  Compute runs in hand-written sm_100a
kernels in libdoublep_b200.so (C ABI: include/doublep_b200.h), loaded with
ctypes; this package is the host-side mirror of the reference interface.
"""

from .cache import (
    Cluster,
    ClusteredCache,
    ClusteredLayer,
    EstimationData,
    KvCache,
    QueryTrace,
    build_clustered_cache,
    cluster_layer,
    default_cluster_count,
    device_cache,
    device_clustered,
    head_seed,
)
from .engine import (
    PRESETS,
    AttentionOutput,
    ClusterEstimate,
    DecodeGraph,
    DecodeWorkspace,
    DoublePConfig,
    SelectionPlan,
    TopPResult,
    build_cache_for_config,
    cluster_topk_attention,
    decode_step,
    dense_attention,
    estimate_cluster_distribution,
    full_attention,
    plan_selection,
    sparse_attention,
)
from .metrics import (
    adaptive_token_budget,
    baseline_cluster_topk,
    baseline_token_topk,
    baseline_token_topp_fixed_budget,
    cluster_approx_error,
    full_attention_weights,
    output_error,
    recovered_mass,
    token_topk_attention,
    token_weights,
    true_token_weights,
    violation_rate,
)

__version__ = "0.1.0"
BACKEND = "b200"

__all__ = [
    "Cluster", "EstimationData", "QueryTrace", "device_cache", "device_clustered", "baseline_cluster_topk",
    "baseline_token_topp_fixed_budget",
    "AttentionOutput", "BACKEND", "ClusterEstimate", "ClusteredCache", "ClusteredLayer", "DecodeGraph", "DecodeWorkspace",
    "DoublePConfig", "KvCache", "PRESETS", "SelectionPlan", "TopPResult", "build_cache_for_config",
    "build_clustered_cache", "cluster_layer", "cluster_topk_attention", "decode_step", "default_cluster_count", "dense_attention",
    "estimate_cluster_distribution", "full_attention", "head_seed", "plan_selection", "sparse_attention",
    "adaptive_token_budget", "baseline_token_topk", "cluster_approx_error", "full_attention_weights",
    "output_error", "recovered_mass", "token_topk_attention", "token_weights", "true_token_weights",
    "violation_rate",
]
