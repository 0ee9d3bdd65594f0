"""CPU oracle for the Double-P decode path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference algorithm
(`/root/reference/pkg/src/doublep`, arxiv 2602.05191, package ``doublep``
0.1.0).  It exists so that the CUDA path can be checked against the
reference semantics on machines where the reference itself is not present
(the GPU box).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker / the timed CPU baseline -- never as part of the
product path (``paper_2602_05191_b200`` never imports this file).

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the real reference (``oracle/gen_golden.py``,
run in the build container where ``/root/reference`` exists) and against
the reference's own known-answer tests.

All accumulation is float64, as in the reference contract
(`kernels.py:6-8`).  Ties go to the lower index everywhere.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# Kernel-level primitives (reference plugin seam, kernels.py:47-96)
# ----------------------------------------------------------------------------


def scaled_logits(keys, q, scale):
    """(keys @ q) * scale in float64 -- `_kernels_py.py:14-18`."""
    return (np.asarray(keys).astype(np.float64, copy=False) @ np.asarray(q, np.float64)) * scale


def logsumexp(x):
    """Max-subtracted LSE, exact for one element -- `_kernels_py.py:29-35`."""
    x = np.asarray(x, dtype=np.float64)
    m = float(np.max(x))
    if x.size == 1:
        return m
    return m + float(np.log(np.sum(np.exp(x - m))))


def softmax(x):
    """Max-subtracted softmax -- `_kernels_py.py:38-42`."""
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(x - np.max(x))
    return e / np.sum(e)


def weighted_sum(w, mat):
    """w @ mat in float64 -- `_kernels_py.py:45-48`."""
    return np.asarray(w, np.float64) @ np.asarray(mat).astype(np.float64, copy=False)


def nearest_centroid(points, centroids):
    """Squared-Euclidean argmin, ties -> lowest index -- `_kernels_py.py:58-77`.

    Uses the |x|^2 - 2x.c + |c|^2 expansion clamped at 0 (the NumPy backend's
    formulation).  Processed in row blocks to bound memory."""
    x = np.asarray(points).astype(np.float64, copy=False)
    c = np.asarray(centroids).astype(np.float64, copy=False)
    cc = np.sum(c * c, axis=1)[None, :]
    n = x.shape[0]
    assign = np.empty(n, dtype=np.int64)
    best = np.empty(n, dtype=np.float64)
    step = max(1, (1 << 24) // max(1, c.shape[0]))
    for s in range(0, n, step):
        xb = x[s:s + step]
        d2 = np.sum(xb * xb, axis=1)[:, None] - 2.0 * (xb @ c.T) + cc
        a = np.argmin(d2, axis=1)
        b = d2[np.arange(xb.shape[0]), a]
        np.maximum(b, 0.0, out=b)
        assign[s:s + step] = a
        best[s:s + step] = b
    return assign, best


def sorted_prefix_count(sorted_probs, p):
    """Early-stop prefix count on a non-increasing vector -- `_kernels_py.py:80-99`."""
    sp = np.asarray(sorted_probs, dtype=np.float64)
    total = 0.0
    prev = np.inf
    for i in range(sp.shape[0]):
        v = sp[i]
        if v > prev:
            raise ValueError("input not sorted")
        prev = v
        total += v
        if total >= p:
            return i + 1
    return sp.shape[0]


def scaled_logits_seq(keys, idx, q, scale):
    """The compiled backend's loop order (`_kernels_cy.pyx:21-50`): per row, a
    float64 running sum over j of keys[row, j] * q[j] (each product and add
    rounded separately), then one multiply by ``scale``.  Vectorised over
    rows; bit-identical to the Cython backend (pinned against its outputs in
    tests/golden/kernels_seam.npz)."""
    keys = np.asarray(keys)
    rows = keys if idx is None else keys[np.asarray(idx, dtype=np.intp)]
    rows = rows.astype(np.float64, copy=False)
    q = np.asarray(q, dtype=np.float64)
    acc = np.zeros(rows.shape[0], dtype=np.float64)
    for j in range(rows.shape[1]):
        acc = acc + rows[:, j] * q[j]
    return acc * scale


def nearest_centroid_direct(points, centroids):
    """The compiled backend's formulation (`_kernels_cy.pyx:115-140`): direct
    differences, float64 running sum over j, strict ``<`` over centroids in
    index order (ties -> lowest index).  Differs from the NumPy backend's
    expansion (:func:`nearest_centroid`) in the last bits of the distance."""
    x = np.asarray(points).astype(np.float64, copy=False)
    c = np.asarray(centroids, dtype=np.float64)
    n = x.shape[0]
    best = np.full(n, np.inf)
    assign = np.zeros(n, dtype=np.int64)
    for ci in range(c.shape[0]):
        dist = np.zeros(n, dtype=np.float64)
        for j in range(x.shape[1]):
            diff = x[:, j] - c[ci, j]
            dist = dist + diff * diff
        better = dist < best
        best = np.where(better, dist, best)
        assign = np.where(better, ci, assign)
    return assign, best


def output_error(candidate, reference):
    """Relative L2 error -- `metrics.py:15-23`."""
    a = candidate.output if isinstance(candidate, AttentionOutput) else np.asarray(candidate)
    b = reference.output if isinstance(reference, AttentionOutput) else np.asarray(reference)
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    denom = max(float(np.linalg.norm(b)), 1e-12)
    return float(np.linalg.norm(a - b)) / denom


# ----------------------------------------------------------------------------
# Selection (selection.py:16-92)
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class TopPResult:
    selected: np.ndarray
    cumulative_mass: float
    p: float


def _desc_order(scores):
    """Stable descending order, lower index first on ties -- `selection.py:30-33`."""
    return np.argsort(-np.asarray(scores, dtype=np.float64), kind="stable")


def top_p_select(probs, p):
    """Minimal descending prefix with cumsum/total >= p -- `selection.py:36-65`."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")
    probs = np.asarray(probs, dtype=np.float64)
    if probs.ndim != 1 or probs.size == 0:
        raise ValueError("probs must be a nonempty 1-D vector")
    if not np.all(np.isfinite(probs)):
        raise ValueError("non-finite probability")
    if np.any(probs < 0.0):
        raise ValueError("negative probability")
    total = float(probs.sum())
    if total <= 0.0:
        raise ValueError("zero total mass")
    order = _desc_order(probs)
    cumulative = np.cumsum(probs[order]) / total
    count = int(np.searchsorted(cumulative, p, side="left")) + 1
    if count > order.size:
        count = order.size
    return TopPResult(selected=order[:count], cumulative_mass=float(cumulative[count - 1]), p=p)


def top_p_select_sorted(sorted_probs, p):
    """`selection.py:68-82`."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")
    sp = np.asarray(sorted_probs, dtype=np.float64)
    if sp.ndim != 1 or sp.size == 0:
        raise ValueError("sorted_probs must be a nonempty 1-D vector")
    return sorted_prefix_count(sp, p)


def top_k_select(scores, k):
    """`selection.py:85-92`."""
    scores = np.asarray(scores, dtype=np.float64)
    if scores.ndim != 1 or scores.size == 0:
        raise ValueError("scores must be a nonempty 1-D vector")
    if not 1 <= k <= scores.size:
        raise ValueError(f"k must be in [1, {scores.size}], got {k}")
    return _desc_order(scores)[:k]


# ----------------------------------------------------------------------------
# Synthetic workload (workload.py:1-194)
# ----------------------------------------------------------------------------

PROFILES = ("peaked", "heavy", "uniform", "mixed")
_TAG_KEYS, _TAG_VALUES, _TAG_QUERIES = 0, 1, 2


@dataclass(frozen=True)
class WorkloadSpec:
    """`workload.py:34-80` (validation restated)."""

    context_len: int
    head_dim: int
    num_layers: int = 1
    num_kv_heads: int = 1
    gqa_group: int = 1
    num_steps: int = 1
    num_blobs: int = 8
    blob_spread: float = 0.3
    blob_separation: float = 1.0
    tail_profile: str = "mixed"
    seed: int = 0
    sink: int = 4
    window: int = 64

    def __post_init__(self):
        if self.tail_profile not in PROFILES:
            raise ValueError(f"unknown tail profile {self.tail_profile!r}")
        for name in ("context_len", "head_dim", "num_layers", "num_kv_heads",
                     "gqa_group", "num_steps", "num_blobs"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.context_len <= self.sink + self.window:
            raise ValueError("context_len must exceed sink + window")

    @property
    def num_query_heads(self):
        return self.num_kv_heads * self.gqa_group


def profile_for_head(spec, layer, query_head):
    """`workload.py:83-88`."""
    if spec.tail_profile != "mixed":
        return spec.tail_profile
    cycle = ("peaked", "heavy", "uniform")
    return cycle[(layer * spec.num_query_heads + query_head) % len(cycle)]


def _rng(spec, tag, layer, head):
    """`workload.py:91-94`."""
    return np.random.default_rng(np.random.SeedSequence([spec.seed, tag, layer, head]))


def _unit(v):
    n = np.linalg.norm(v)
    return v if n == 0.0 else v / n


def _multi_blob_direction(centers, chosen):
    """`workload.py:104-127`."""
    dim = centers.shape[1]
    chosen = list(chosen)
    suppressed = []
    while True:
        rows = centers[chosen + suppressed]
        targets = np.concatenate([np.ones(len(chosen)), np.zeros(len(suppressed))])
        u, *_ = np.linalg.lstsq(rows, targets, rcond=None)
        u = _unit(u)
        level = float(np.mean(centers[chosen] @ u))
        taken = set(chosen) | set(suppressed)
        others = [b for b in range(len(centers)) if b not in taken]
        if not others or len(taken) >= dim - 2:
            return u
        leaks = centers[others] @ u
        worst = int(np.argmax(leaks))
        if leaks[worst] <= 0.55 * level:
            return u
        suppressed.append(others[worst])


def _peaked_query(rng, centers, spec):
    """`workload.py:130-142`."""
    if rng.random() < 0.25:
        count = min(max(2, spec.num_blobs // 3), len(centers))
        chosen = rng.choice(len(centers), size=count, replace=False)
        direction = _multi_blob_direction(centers, chosen)
    else:
        direction = _unit(centers[int(rng.integers(len(centers)))])
    gain = 3.0 * rng.uniform(1.0, 1.3)
    return gain * np.sqrt(spec.head_dim) * direction


def _heavy_query(rng, centers, spec):
    """`workload.py:145-151`."""
    count = min(max(2, spec.num_blobs // 4), len(centers))
    chosen = rng.choice(len(centers), size=count, replace=False)
    direction = _unit(np.sum([_unit(centers[b]) for b in chosen], axis=0))
    gain = 3.7 * rng.uniform(0.75, 1.25)
    return gain * np.sqrt(spec.head_dim) * direction


def generate_head(spec, layer, head):
    """Keys/values/blob centres of one (layer, kv head) -- `workload.py:160-173`."""
    n, d = spec.context_len, spec.head_dim
    rng = _rng(spec, _TAG_KEYS, layer, head)
    c = rng.normal(0.0, spec.blob_separation, size=(spec.num_blobs, d))
    assignment = rng.integers(0, spec.num_blobs, size=n)
    keys = (c[assignment] + rng.normal(0.0, spec.blob_spread, size=(n, d))).astype(np.float32)
    vrng = _rng(spec, _TAG_VALUES, layer, head)
    vcenters = vrng.normal(0.0, 1.0, size=(spec.num_blobs, d))
    values = (vcenters[assignment] + vrng.normal(0.0, 0.5, size=(n, d))).astype(np.float32)
    return keys, values, c


def generate_queries(spec, layer, qhead, centers):
    """All steps of one (layer, q head) -- `workload.py:178-190`."""
    d = spec.head_dim
    rng = _rng(spec, _TAG_QUERIES, layer, qhead)
    profile = profile_for_head(spec, layer, qhead)
    out = np.empty((spec.num_steps, d), dtype=np.float32)
    for step in range(spec.num_steps):
        if profile == "peaked":
            q = _peaked_query(rng, centers, spec)
        elif profile == "heavy":
            q = _heavy_query(rng, centers, spec)
        else:
            q = np.zeros(d)
        out[step] = q.astype(np.float32)
    return out


def generate(spec):
    """Returns (keys, values, queries, gqa_group) -- `workload.py:154-194`.

    keys/values f32[L,Hkv,N,d]; queries f32[S,L,Hq,d]."""
    n, d = spec.context_len, spec.head_dim
    keys = np.empty((spec.num_layers, spec.num_kv_heads, n, d), dtype=np.float32)
    values = np.empty_like(keys)
    centers = {}
    for layer in range(spec.num_layers):
        for head in range(spec.num_kv_heads):
            k, v, c = generate_head(spec, layer, head)
            keys[layer, head], values[layer, head] = k, v
            centers[layer, head] = c
    queries = np.empty((spec.num_steps, spec.num_layers, spec.num_query_heads, d), dtype=np.float32)
    for layer in range(spec.num_layers):
        for qh in range(spec.num_query_heads):
            queries[:, layer, qh] = generate_queries(spec, layer, qh, centers[layer, qh // spec.gqa_group])
    return keys, values, queries


# ----------------------------------------------------------------------------
# k-means clustering (clustering.py:36-107)
# ----------------------------------------------------------------------------


def head_seed(seed, layer, head):
    """Per-head k-means seed -- `clustering.py:295`."""
    return int(np.random.SeedSequence([seed, layer, head]).generate_state(1)[0])


def plusplus_init(x64, k, rng):
    """k-means++ seeding -- `clustering.py:36-55`.

    `rng.choice(n, p=dsq/total)` is restated as NumPy's Generator.choice does
    it: cdf = cumsum(p); cdf /= cdf[-1]; searchsorted(cdf, rng.random(),
    side='right').  Returns (centers f64[k,d], picked indices i64[k])."""
    n = x64.shape[0]
    centers = np.empty((k, x64.shape[1]), dtype=np.float64)
    picks = np.empty(k, dtype=np.int64)
    first = int(rng.integers(n))
    centers[0] = x64[first]
    picks[0] = first
    if k == 1:
        return centers, picks
    dsq = np.sum((x64 - centers[0]) ** 2, axis=1)
    for i in range(1, k):
        total = float(dsq.sum())
        if total > 0.0:
            cdf = (dsq / total).cumsum()
            cdf /= cdf[-1]
            idx = int(cdf.searchsorted(rng.random(), side="right"))
        else:
            idx = int(rng.integers(n))
        centers[i] = x64[idx]
        picks[i] = idx
        np.minimum(dsq, np.sum((x64 - centers[i]) ** 2, axis=1), out=dsq)
    return centers, picks


def init_stream(seed, n, k):
    """The host-side RNG stream a replayed k-means++ consumes, assuming no
    degenerate (total == 0) step: (first index, uniforms f64[k-1])."""
    rng = np.random.default_rng(seed)
    first = int(rng.integers(n))
    u = rng.random(k - 1) if k > 1 else np.empty(0)
    return first, u


@dataclass
class KMeansResult:
    assignments: np.ndarray
    centroids: np.ndarray
    objective: list
    iterations: int = 0


def lloyd(x, centroids, max_iters):
    """Lloyd loop with empty-cluster drop -- `clustering.py:81-107`."""
    x64 = np.asarray(x).astype(np.float64, copy=False)
    centroids = np.array(centroids, dtype=np.float64, copy=True)
    objective = []
    prev_assign = None
    assign = None
    iters = 0
    for _ in range(max_iters):
        iters += 1
        assign, sqdist = nearest_centroid(x, centroids)
        objective.append(float(sqdist.sum()))
        used = np.unique(assign)
        dropped = used.size < centroids.shape[0]
        if dropped:
            remap = np.full(centroids.shape[0], -1, dtype=np.int64)
            remap[used] = np.arange(used.size)
            assign = remap[assign]
            centroids = centroids[used]
        if not dropped and prev_assign is not None and np.array_equal(assign, prev_assign):
            break
        prev_assign = assign
        centroids = _means(x64, assign, centroids.shape[0])
    final = _means(x64, assign, centroids.shape[0])
    return KMeansResult(assignments=assign, centroids=final, objective=objective, iterations=iters)


def _means(x64, assign, k):
    sums = np.zeros((k, x64.shape[1]))
    np.add.at(sums, assign, x64)
    cnt = np.bincount(assign, minlength=k).astype(np.float64)
    return sums / cnt[:, None]


def kmeans_fit(keys, k, max_iters=25, seed=0):
    """`clustering.py:58-107`."""
    keys = np.asarray(keys)
    if keys.ndim != 2 or keys.shape[0] < 1:
        raise ValueError("keys must be a nonempty (n, d) matrix")
    n = keys.shape[0]
    if k < 1:
        raise ValueError("cluster count must be >= 1")
    if k > n:
        raise ValueError(f"more clusters than points: k={k}, n={n}")
    x64 = keys.astype(np.float64, copy=False)
    rng = np.random.default_rng(seed)
    centroids, _ = plusplus_init(x64, k, rng)
    return lloyd(keys, centroids, max_iters)


def default_cluster_count(middle_len, tokens_per_cluster=32):
    """`clustering.py:261-263`."""
    return max(1, math.ceil(middle_len / tokens_per_cluster))


# ----------------------------------------------------------------------------
# Cluster tables (the device layout, restated on the host for checking)
# ----------------------------------------------------------------------------


@dataclass
class HeadTables:
    """One (layer, kv head) clustered view, the oracle's mirror of the device
    tables: clusters in compacted k-means id order (`clustering.py:300-311`),
    then residual singletons (`clustering.py:219-229`).

    members[c] : int64 ascending token positions
    centroids  : f64[K,d]  (exact fp64 means, or the device's fp32 values)
    value_means: f64[K,d]
    """

    members: list
    centroids: np.ndarray
    value_means: np.ndarray

    @property
    def sizes(self):
        return np.array([m.size for m in self.members], dtype=np.int64)

    @property
    def log_sizes(self):
        return np.log(self.sizes.astype(np.float64))


def build_head_tables(keys_h, values_h, k, sink, window, max_iters=25, seed_for_head=0):
    """`build_clustered_cache` for one head -- `clustering.py:266-314`."""
    n = keys_h.shape[0]
    start, stop = sink, n - window
    fit = kmeans_fit(keys_h[start:stop], k, max_iters=max_iters, seed=seed_for_head)
    values64 = values_h[start:stop].astype(np.float64)
    members, vmeans = [], []
    for c in range(fit.centroids.shape[0]):
        local = np.flatnonzero(fit.assignments == c)
        vsum = values64[local].sum(axis=0)
        members.append((local + start).astype(np.int64))
        vmeans.append(vsum / local.size)
    return HeadTables(members=members, centroids=fit.centroids, value_means=np.asarray(vmeans)), fit


def clamp_k(n, sink, window, k=None, tokens_per_cluster=32):
    """Cluster-count policy -- `clustering.py:276-288`."""
    if sink < 0 or window < 0:
        raise ValueError("sink and window must be >= 0")
    middle = n - window - sink
    if middle < 1:
        raise ValueError(f"no middle tokens to cluster: sink {sink} + window {window} >= context {n}")
    if k is None:
        k = default_cluster_count(middle, tokens_per_cluster)
    if k < 1:
        raise ValueError("cluster count must be >= 1")
    return min(k, middle)


# ----------------------------------------------------------------------------
# Decode step (engine.py:158-278)
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class AttentionOutput:
    output: np.ndarray
    normalizer: float
    exact_token_count: int
    approx_cluster_count: int
    log_normalizer: float = 0.0


@dataclass
class Estimate:
    log_masses: np.ndarray
    probs: np.ndarray
    order: np.ndarray


@dataclass
class Plan:
    stage1: TopPResult
    exact_clusters: np.ndarray
    approx_clusters: np.ndarray
    exact_tokens: np.ndarray


def estimate(q, tables, d):
    """`engine.py:158-177`."""
    if len(tables.members) == 0:
        raise ValueError("no clusters for this head")
    lm = scaled_logits(tables.centroids, q, 1.0 / np.sqrt(d)) + tables.log_sizes
    probs = softmax(lm)
    return Estimate(log_masses=lm, probs=probs, order=np.argsort(-probs, kind="stable"))


def plan(est, tables, p1, p2, sink_idx, window_idx):
    """`engine.py:180-213`."""
    stage1 = top_p_select(est.probs, p1)
    cp = stage1.selected
    n2 = len(top_p_select(est.probs[cp], p2).selected)
    exact = cp[:n2]
    approx = cp[n2:]
    tokens = np.concatenate([sink_idx, window_idx, *[tables.members[int(i)] for i in exact]])
    tokens.sort()
    return Plan(stage1=stage1, exact_clusters=exact, approx_clusters=approx, exact_tokens=tokens)


def mixed_attention(q, keys_h, values_h, tables, exact_tokens, approx_clusters, est):
    """`engine.py:216-252`; keys_h/values_h are the full-position rows."""
    d = keys_h.shape[1]
    scale = 1.0 / np.sqrt(d)
    exact_tokens = np.asarray(exact_tokens, dtype=np.int64)
    approx_clusters = np.asarray(approx_clusters, dtype=np.int64)
    exact_logits = scaled_logits(keys_h[exact_tokens], q, scale)
    combined = np.concatenate([exact_logits, est.log_masses[approx_clusters]])
    log_z = logsumexp(combined)
    w = np.exp(combined - log_z)
    out = np.zeros(d, dtype=np.float64)
    if exact_tokens.size:
        out += weighted_sum(w[: exact_tokens.size], values_h[exact_tokens])
    if approx_clusters.size:
        out += weighted_sum(w[exact_tokens.size:], tables.value_means[approx_clusters])
    return AttentionOutput(output=out, normalizer=float(np.exp(log_z)),
                           exact_token_count=int(exact_tokens.size),
                           approx_cluster_count=int(approx_clusters.size), log_normalizer=log_z)


def decode_step(q, keys_h, values_h, tables, p1, p2, sink, window):
    """`engine.py:267-278` for one (q head -> kv head)."""
    n = keys_h.shape[0]
    est = estimate(q, tables, keys_h.shape[1])
    pl = plan(est, tables, p1, p2, np.arange(sink, dtype=np.int64),
              np.arange(n - window, n, dtype=np.int64))
    out = mixed_attention(q, keys_h, values_h, tables, pl.exact_tokens, pl.approx_clusters, est)
    return out, pl, est


def cluster_topk(q, keys_h, values_h, tables, budget, sink, window):
    """Fixed cluster-budget baseline -- `engine.py:318-338`: the `budget`
    clusters of largest estimated mass exact (plus sink and window), every
    other cluster approximated, one normaliser."""
    n = keys_h.shape[0]
    est = estimate(q, tables, keys_h.shape[1])
    if not 1 <= budget <= est.probs.size:
        raise ValueError(f"cluster budget must be in [1, {est.probs.size}], got {budget}")
    chosen = est.order[:budget]
    rest = est.order[budget:]
    tokens = np.concatenate([np.arange(sink, dtype=np.int64), np.arange(n - window, n, dtype=np.int64),
                             *[tables.members[int(i)] for i in chosen]])
    tokens.sort()
    return mixed_attention(q, keys_h, values_h, tables, tokens, rest, est)


def full_attention(q, keys_h, values_h):
    """Dense oracle -- `engine.py:122-144`."""
    d = keys_h.shape[1]
    logits = scaled_logits(keys_h, q, 1.0 / np.sqrt(d))
    lse = logsumexp(logits)
    w = np.exp(logits - lse)
    return AttentionOutput(output=weighted_sum(w, values_h), normalizer=float(np.exp(lse)),
                           exact_token_count=keys_h.shape[0], approx_cluster_count=0,
                           log_normalizer=lse)


# ----------------------------------------------------------------------------
# Measurement side: token top-k baseline and metrics (engine.py:293-315,
# metrics.py:26-76)
# ----------------------------------------------------------------------------


def full_attention_weights(q, keys_h):
    """`engine.py:122-132`: (weights f64[N], lse)."""
    logits = scaled_logits(keys_h, q, 1.0 / np.sqrt(keys_h.shape[1]))
    lse = logsumexp(logits)
    return np.exp(logits - lse), lse


def token_topk(q, keys_h, values_h, budget):
    """`engine.py:293-315` baseline_token_topk: exact attention over the
    `budget` tokens of largest true weight, renormalised over the subset.
    Returns (AttentionOutput, captured, idx)."""
    n = keys_h.shape[0]
    if not 1 <= budget <= n:
        raise ValueError(f"budget must be in [1, {n}], got {budget}")
    w, lse = full_attention_weights(q, keys_h)
    idx = top_k_select(w, budget)
    captured = float(w[idx].sum())
    out = weighted_sum(w[idx] / captured, values_h[idx])
    return (AttentionOutput(output=out, normalizer=float(np.exp(lse)) * captured, exact_token_count=int(budget),
                            approx_cluster_count=0, log_normalizer=lse + math.log(captured)), captured, idx)


def recovered_mass(w, exact_tokens):
    """`metrics.py:26-39`: true mass of a plan's exact tokens."""
    return float(w[np.asarray(exact_tokens, dtype=np.int64)].sum())


def adaptive_token_budget(w, p):
    """`metrics.py:41-50`: minimal token count whose true mass reaches p."""
    order = np.argsort(-w, kind="stable")
    cum = np.cumsum(w[order])
    return int(np.searchsorted(cum, p, side="left") + 1)


def violation_rate(recovered, p):
    """`metrics.py:53-58`."""
    arr = np.asarray(recovered, dtype=np.float64)
    if arr.size == 0:
        raise ValueError("no recovered masses given")
    return float(np.mean(arr < p))


def cluster_approx_error(w, lse, est, tables):
    """`metrics.py:61-76`: |true mass - exp(log_mass - lse)| per cluster, in
    estimated-rank order.  Returns (errors, order)."""
    true_mass = np.array([w[m].sum() for m in tables.members], dtype=np.float64)
    errors = np.abs(true_mass - np.exp(est.log_masses - lse))
    return errors[est.order], est.order


# ----------------------------------------------------------------------------
# Decode-time growth (clustering.py:170-229) and split-KV merge
# ----------------------------------------------------------------------------


def grow_tables(base, keys_h_full, values_h_full, context_len, total_tokens, window):
    """Residual singleton pool after appends -- `clustering.py:178-229`.

    keys_h_full/values_h_full hold all total_tokens positions."""
    members = list(base.members)
    cents = [base.centroids]
    vms = [base.value_means]
    res = list(range(context_len - window, total_tokens - window))
    for pos in res:
        members.append(np.array([pos], dtype=np.int64))
    if res:
        cents.append(keys_h_full[res].astype(np.float64))
        vms.append(values_h_full[res].astype(np.float64))
    return HeadTables(members=members, centroids=np.concatenate(cents), value_means=np.concatenate(vms))


def lse_merge(ms, ls, os_):
    """Combine split partials (m, l, o): M = max m, L = sum l e^(m-M),
    o = sum l e^(m-M) o / L.  Empty partials carry m=-inf, l=0."""
    ms = np.asarray(ms, np.float64)
    ls = np.asarray(ls, np.float64)
    os_ = np.asarray(os_, np.float64)
    M = np.max(ms)
    if not np.isfinite(M):
        return -np.inf, 0.0, np.zeros(os_.shape[-1])
    w = ls * np.exp(ms - M)
    L = w.sum()
    return M, L, (w[:, None] * os_).sum(axis=0) / L
