"""Device-resident clustered KV cache (the B200 layout of ClusteredCache).

Reference: /root/reference/pkg/src/doublep/clustering.py:140-314 and
kvcache.py:50-139.  One ``ClusteredLayer`` holds one layer of a batch of
sequences in the cluster-contiguous layout described in
include/doublep_b200.h; ``ClusteredCache`` mirrors the reference's
per-(layer, kv head) object for a single sequence and wraps one
``ClusteredLayer`` per layer.

Clustering runs on the GPU (libdoublep_b200.so: dp_cluster_build).  The host
only replays the reference's RNG stream (numpy PCG64, clustering.py:78,295)
so the k-means++ seeding picks the same points as the reference.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N

DEFAULT_TOKENS_PER_CLUSTER = 32
DEFAULT_MAX_ITERS = 25

_DT = {torch.float32: N.DP_F32, torch.bfloat16: N.DP_BF16}


def dtype_code(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}; expected float32 or bfloat16") from None


def default_cluster_count(middle_len, tokens_per_cluster=DEFAULT_TOKENS_PER_CLUSTER):
    """`clustering.py:261-263`."""
    return max(1, math.ceil(middle_len / tokens_per_cluster))


def pad_dim(t, width=None):
    """Zero-pad the last axis to ``width`` (default: the next multiple of 8,
    the kernels' 16-B row granule).  Zero key/query coordinates leave every
    dot product and distance unchanged; padded value coordinates stay 0."""
    d = t.shape[-1]
    width = ((d + 7) // 8) * 8 if width is None else width
    if width == d:
        return t
    return torch.nn.functional.pad(t, (0, width - d))


def head_seed(seed, layer, head, seq=0):
    """Per-head k-means seed, `clustering.py:295` (seq > 0 extends the
    reference's single-sequence key with the batch index)."""
    key = [seed, layer, head] if seq == 0 else [seed, layer, head, seq]
    return int(np.random.SeedSequence(key).generate_state(1)[0])


def rng_stream(seed, n, k, degenerate_from=None):
    """The draws `_plusplus_init` consumes (`clustering.py:41-52`):
    first = rng.integers(n), then one rng.random() per further centre, or
    rng.integers(n) from the first zero-mass step on."""
    rng = np.random.default_rng(seed)
    first = int(rng.integers(n))
    stop = k if degenerate_from is None else min(int(degenerate_from), k)
    u = np.zeros(max(k - 1, 0))
    alt = np.zeros(max(k - 1, 0), dtype=np.int32)
    if stop > 1:
        u[: stop - 1] = rng.random(stop - 1)  # same bits as stop-1 scalar draws
    for i in range(stop, k):
        alt[i - 1] = int(rng.integers(n))
    return first, u, alt


def _check_geometry(n, sink, window, k, tokens_per_cluster):
    """`clustering.py:276-288`."""
    if sink < 0 or window < 0:
        raise ValueError("sink and window must be >= 0")
    middle = n - window - sink
    if middle < 1:
        raise ValueError(f"no middle tokens to cluster: sink {sink} + window {window} >= context {n}")
    if k is None:
        k = default_cluster_count(middle, tokens_per_cluster)
    if k < 1:
        raise ValueError("cluster count must be >= 1")
    return min(k, middle), middle


class ClusteredLayer:
    """One layer, batch of B sequences, all kv heads, in the device layout.

    keys/values [B,H,row_cap,d]; offs [B,H,cap+1]; nclusters [B,H];
    centroids/value_means fp32 [B,H,cap,d]; perm [B,H,row_cap] (original
    position of every row, for parity/reporting only)."""

    def __init__(self, keys, values, offs, nclusters, centroids, value_means, perm, n_tokens, sink,
                 window, objective=None, iters=None, prefill_tokens=None, logical_dim=None):
        self.keys, self.values = keys, values
        # head_dim of the caller's vectors when the device rows are zero-padded
        # to a multiple of 8 (pad_dim); scores use 1/sqrt(logical_dim)
        self.logical_dim = int(logical_dim) if logical_dim is not None else None
        self.offs, self.nclusters = offs, nclusters
        self.centroids, self.value_means = centroids, value_means
        self.perm = perm
        self.n_tokens = int(n_tokens)
        self.prefill_tokens = int(prefill_tokens if prefill_tokens is not None else n_tokens)
        self.sink, self.window = int(sink), int(window)
        self.objective, self.iters = objective, iters
        self._keep = None

    # geometry -----------------------------------------------------------
    @property
    def batch(self):
        return self.keys.shape[0]

    @property
    def kv_heads(self):
        return self.keys.shape[1]

    @property
    def row_cap(self):
        return self.keys.shape[2]

    @property
    def head_dim(self):
        return self.keys.shape[3]

    @property
    def dim(self):
        """Head dim of the caller's vectors (== head_dim unless padded)."""
        return self.logical_dim if self.logical_dim is not None else self.keys.shape[3]

    @property
    def attn_scale(self):
        return 1.0 / math.sqrt(self.dim)

    @property
    def cluster_cap(self):
        return self.centroids.shape[2]

    @property
    def dtype(self):
        return self.keys.dtype

    @property
    def device(self):
        return self.keys.device

    def view(self, b=None, h=None):
        """dp_cache_view over the whole layer, or over one (b, h) head.  The
        whole-layer view is cached (the step path calls this every layer) and
        rebuilt when the token count changes."""
        if b is None:
            cv = self.__dict__.get("_view")
            if cv is not None and cv.n_tokens == self.n_tokens:
                return cv
            self.__dict__["_view"] = cv = self._make_view(None, None)
            return cv
        return self._make_view(b, h)

    def _make_view(self, b, h):
        v = N.CacheView()
        v.batch, v.kv_heads = self.batch, self.kv_heads
        v.head_dim, v.dtype = self.head_dim, dtype_code(self.keys)
        v.row_cap, v.n_tokens = self.row_cap, self.n_tokens
        v.sink, v.window, v.cluster_cap = self.sink, self.window, self.cluster_cap
        k, vv, o, nc, c, vb = self.keys, self.values, self.offs, self.nclusters, self.centroids, self.value_means
        if b is not None:
            k, vv, o, nc, c, vb = (t[b:b + 1, h:h + 1] for t in (k, vv, o, nc, c, vb))
            v.batch = v.kv_heads = 1
        v.keys, v.values = k.data_ptr(), vv.data_ptr()
        v.offs, v.nclusters = o.data_ptr(), nc.data_ptr()
        v.centroids, v.value_means = c.data_ptr(), vb.data_ptr()
        return v

    # decode-time growth -------------------------------------------------
    def append(self, new_k, new_v, stream=None):
        """Append one token per (b, h) (`ClusteredCache.append_tokens`,
        clustering.py:182-196).  new_k/new_v [B,H,d] on device."""
        want = (self.batch, self.kv_heads, self.dim)
        if tuple(new_k.shape) != want or tuple(new_v.shape) != want:
            raise ValueError(f"appended token must have shape {want}")
        new_k, new_v = pad_dim(new_k, self.head_dim), pad_dim(new_v, self.head_dim)
        # the reference grows without bound (clustering.py:182-196): when the
        # rows or the cluster table are full, reallocate with headroom (the
        # `growth` argument of build_clustered_cache pre-reserves it instead)
        need_c = self._prefill_k + (self.n_tokens + 1 - self.prefill_tokens)
        if self.n_tokens >= self.row_cap or \
                (self.n_tokens - self.window >= self.sink and need_c > self.cluster_cap):
            step = max(64, self.row_cap // 8)
            self.reserve(self.n_tokens + step, max(self.cluster_cap, need_c + step))
        nk = new_k.to(self.dtype).contiguous()
        nv = new_v.to(self.dtype).contiguous()
        v = self.view()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        N.check(N.lib().dp_append_token(v, N.ptr(nk), N.ptr(nv), st.cuda_stream))
        self.n_tokens += 1
        self._keep = (nk, nv)

    _prefill_k = 0

    def reserve(self, row_cap, cluster_cap):
        """Grow the row and cluster capacity (copies the used part; views and
        captured DecodeGraphs over the old storage become stale)."""
        B, H, R, d = self.keys.shape
        row_cap, cluster_cap = max(int(row_cap), R), max(int(cluster_cap), self.cluster_cap)
        if row_cap == R and cluster_cap == self.cluster_cap:
            return
        n = self.n_tokens

        def grow(t, size, dim, fill=0):
            shape = list(t.shape)
            shape[dim] = size
            out = torch.full(shape, fill, dtype=t.dtype, device=t.device)
            out.narrow(dim, 0, t.shape[dim]).copy_(t)
            return out

        k = torch.empty((B, H, row_cap, d), dtype=self.keys.dtype, device=self.device)
        v = torch.empty_like(k)
        k[:, :, :n].copy_(self.keys[:, :, :n])
        v[:, :, :n].copy_(self.values[:, :, :n])
        self.keys, self.values = k, v
        self.offs = grow(self.offs, cluster_cap + 1, 2)
        self.centroids = grow(self.centroids, cluster_cap, 2)
        self.value_means = grow(self.value_means, cluster_cap, 2)
        if self.perm is not None:
            self.perm = grow(self.perm, row_cap, 2)
        self.__dict__.pop("_view", None)

    def split(self):
        """One single-sequence ClusteredLayer per batch entry, sharing storage
        (used to cluster many layers in one launch, then hand them out)."""
        out = []
        for b in range(self.batch):
            sl = lambda t: None if t is None else t[b:b + 1]  # noqa: E731
            lay = ClusteredLayer(sl(self.keys), sl(self.values), sl(self.offs), sl(self.nclusters),
                                 sl(self.centroids), sl(self.value_means), sl(self.perm), self.n_tokens,
                                 self.sink, self.window, prefill_tokens=self.prefill_tokens,
                                 logical_dim=self.logical_dim)
            lay._prefill_k = self._prefill_k
            out.append(lay)
        return out

    def head(self, b, h):
        """Single-(sequence, kv head) ClusteredLayer sharing this layer's storage."""
        sl = lambda t: None if t is None else t[b:b + 1, h:h + 1]  # noqa: E731
        lay = ClusteredLayer(sl(self.keys), sl(self.values), sl(self.offs), sl(self.nclusters), sl(self.centroids),
                             sl(self.value_means), sl(self.perm), self.n_tokens, self.sink, self.window,
                             prefill_tokens=self.prefill_tokens, logical_dim=self.logical_dim)
        lay._prefill_k = self._prefill_k
        return lay

    # host views for parity ----------------------------------------------
    def head_tables(self, b, h):
        """Host copy of one head's tables (synchronises).  Returns dict with
        members (list of int64 position arrays, cluster order), centroids f64,
        value_means f64, sizes."""
        K = int(self.nclusters[b, h].item())
        offs = self.offs[b, h, :K + 1].cpu().numpy().astype(np.int64)
        perm = self.perm[b, h].cpu().numpy().astype(np.int64)
        members = []
        for c in range(K):
            rows = np.arange(offs[c], offs[c + 1])
            pos = np.where(rows < self.prefill_tokens - self.window, perm[np.minimum(rows, len(perm) - 1)], rows)
            members.append(np.sort(pos))
        return {
            "members": members,
            "centroids": self.centroids[b, h, :K, :self.dim].double().cpu().numpy(),
            "value_means": self.value_means[b, h, :K, :self.dim].double().cpu().numpy(),
            "sizes": np.diff(offs),
            "offs": offs,
        }


def cluster_layer(keys, values, *, k=None, sink=4, window=64, seed=0, max_iters=DEFAULT_MAX_ITERS,
                  tokens_per_cluster=DEFAULT_TOKENS_PER_CLUSTER, layer=0, fp64_assign=True, row_cap=None,
                  extra_clusters=0, stream=None, head_seeds=None, tensor_cores=None):
    """k-means-cluster one layer of a batch on the GPU (`build_clustered_cache`
    for one layer, clustering.py:266-314).  keys/values: CUDA [B,H,N,d] f32
    or bf16 in position order.  ``row_cap``/``extra_clusters`` reserve room
    for decode-time growth.  ``tensor_cores`` (default: wherever it applies --
    bf16 keys, d 64/128, k <= 4096, not fp64 mode) runs the Lloyd assignment
    on tcgen05 with an fp64 re-score of each winner, which reproduces the fp64
    path's assignments and objective."""
    if keys.dim() != 4 or keys.shape != values.shape:
        raise ValueError("keys/values must have shape (batch, kv_heads, context, dim)")
    if keys.dtype != values.dtype:
        raise ValueError("keys/values dtype mismatch")
    B, H, n, d = keys.shape
    k, middle = _check_geometry(n, sink, window, k, tokens_per_cluster)
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    dev = keys.device
    keys = keys.contiguous()
    values = values.contiguous()
    row_cap = n if row_cap is None else max(row_cap, n)
    cap = k + int(extra_clusters)
    p = N.ClusterParams()
    p.batch, p.kv_heads, p.head_dim, p.dtype = B, H, d, dtype_code(keys)
    p.n_tokens, p.sink, p.window, p.k = n, sink, window, k
    if tensor_cores is None:  # the fast path wherever it applies (fp64 mode stays on DFMA)
        tensor_cores = (not fp64_assign and keys.dtype == torch.bfloat16 and d in (64, 128) and k <= 4096
                        and middle >= 128)
    p.max_iters, p.fp64_assign = max_iters, 2 if tensor_cores else int(bool(fp64_assign))

    def streams(degen=None):
        firsts = np.zeros(B * H, dtype=np.int32)
        us = np.zeros((B * H, max(k - 1, 1)))
        alts = np.zeros((B * H, max(k - 1, 1)), dtype=np.int32)
        for b in range(B):
            for h in range(H):
                i = b * H + h
                hs = head_seed(seed, layer, h, b) if head_seeds is None else int(head_seeds[b][h])
                f, u, a = rng_stream(hs, middle, k,
                                     None if degen is None else int(degen[i]))
                firsts[i] = f
                us[i, :k - 1] = u
                alts[i, :k - 1] = a
        return firsts, us, alts

    firsts, us, alts = streams()
    f_d = torch.from_numpy(firsts).to(dev)
    u_d = torch.from_numpy(us).to(dev)
    a_d = torch.from_numpy(alts).to(dev)
    degen = torch.full((B * H,), k, dtype=torch.int32, device=dev)
    opts_i = dict(dtype=torch.int32, device=dev)
    dk = torch.empty((B, H, row_cap, d), dtype=keys.dtype, device=dev)
    dv = torch.empty_like(dk)
    offs = torch.zeros((B, H, cap + 1), **opts_i)
    ncl = torch.zeros((B, H), **opts_i)
    cents = torch.zeros((B, H, cap, d), dtype=torch.float32, device=dev)
    vbar = torch.zeros_like(cents)
    perm = torch.zeros((B, H, row_cap), **opts_i)
    obj = torch.zeros((B * H, max_iters), dtype=torch.float64, device=dev)
    iters = torch.zeros((B * H,), **opts_i)
    ws = torch.empty((N.lib().dp_cluster_workspace_bytes(p),), dtype=torch.uint8, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)

    def run():
        N.check(N.lib().dp_cluster_build(
            p, N.ptr(keys), N.ptr(values), N.ptr(f_d), N.ptr(u_d), N.ptr(a_d), N.ptr(degen), N.ptr(dk),
            N.ptr(dv), row_cap, N.ptr(offs), N.ptr(ncl), N.ptr(cents), N.ptr(vbar), cap, N.ptr(perm),
            N.ptr(obj), N.ptr(iters), N.ptr(ws), ws.numel(), st.cuda_stream))

    run()
    # rare degenerate seeding (all points already centres): the reference then
    # draws rng.integers instead of rng.random; replay that stream and rerun.
    dg = degen.cpu().numpy()
    if np.any(dg < k):
        firsts, us, alts = streams(dg)
        f_d.copy_(torch.from_numpy(firsts))
        u_d.copy_(torch.from_numpy(us))
        a_d.copy_(torch.from_numpy(alts))
        degen.copy_(torch.from_numpy(dg))
        run()
    if window > 0 or sink > 0:
        # rows >= prefill middle keep their own positions
        pass
    lay = ClusteredLayer(dk, dv, offs, ncl, cents, vbar, perm, n, sink, window, objective=obj, iters=iters,
                         prefill_tokens=n)
    lay._prefill_k = k
    return lay


# ---------------------------------------------------------------------------
# reference-signature containers (kvcache.py:50-139, clustering.py:110-314)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class KvCache:
    """Dense per-(layer, kv-head) keys/values (`kvcache.py:50-89`).
    keys/values: [L, Hkv, N, d] numpy or torch; stored on the device."""

    keys: torch.Tensor
    values: torch.Tensor

    def __post_init__(self):
        k = torch.as_tensor(self.keys)
        v = torch.as_tensor(self.values)
        if k.dim() != 4:
            raise ValueError("keys must have shape (layers, kv_heads, context, dim)")
        if k.shape != v.shape:
            raise ValueError(f"keys/values shape mismatch: {tuple(k.shape)} vs {tuple(v.shape)}")
        if min(k.shape) < 1:
            raise ValueError(f"all cache dimensions must be positive, got {tuple(k.shape)}")
        if k.dtype not in (torch.float32, torch.bfloat16):
            k, v = k.float(), v.float()
        if not (torch.isfinite(k.float()).all() and torch.isfinite(v.float()).all()):
            raise ValueError("non-finite entries in keys/values")
        dev = torch.device("cuda")
        object.__setattr__(self, "_dim", int(k.shape[3]))
        object.__setattr__(self, "keys", pad_dim(k.to(dev)).contiguous())
        object.__setattr__(self, "values", pad_dim(v.to(dev)).contiguous())

    @property
    def num_layers(self):
        return self.keys.shape[0]

    @property
    def num_kv_heads(self):
        return self.keys.shape[1]

    @property
    def context_len(self):
        return self.keys.shape[2]

    @property
    def head_dim(self):
        return self._dim

    @property
    def padded_dim(self):
        """Row width on the device (head_dim rounded up to a multiple of 8)."""
        return self.keys.shape[3]


# device copies of foreign caches (the reference's numpy KvCache or any object
# with 4-D .keys/.values), keyed by identity and dropped with the object
_DEV_CACHES = {}


def device_cache(cache):
    """This package's KvCache for ``cache``: itself, or a device copy of any
    object exposing [L, Hkv, N, d] ``keys`` / ``values`` (the reference's
    KvCache, kvcache.py:50-89), made once per object."""
    if isinstance(cache, KvCache):
        return cache
    if not (hasattr(cache, "keys") and hasattr(cache, "values")):
        if isinstance(cache, (tuple, list)) and len(cache) == 2:
            return KvCache(*cache)
        raise TypeError(f"expected a KvCache (an object with .keys and .values), got {type(cache).__name__}")
    key = id(cache)
    hit = _DEV_CACHES.get(key)
    if hit is not None and hit[0]() is cache:
        return hit[1]
    dev = KvCache(cache.keys, cache.values)
    try:
        ref = weakref.ref(cache, lambda _r, k=key: _DEV_CACHES.pop(k, None))
    except TypeError:  # not weak-referenceable: convert per call
        return dev
    _DEV_CACHES[key] = (ref, dev)
    return dev


@dataclass(frozen=True)
class QueryTrace:
    """Per-step decode queries for every layer and query head (`kvcache.py:92-139`).

    queries: [steps, layers, q_heads, d] (numpy or torch, any float dtype;
    kept float32 on the host as in the reference); query head h reads kv
    head h // gqa_group.  ``step_queries`` hands the product path one
    (step, layer) slice as a device tensor [1, q_heads, d]."""

    queries: np.ndarray
    gqa_group: int

    def __post_init__(self):
        q = self.queries
        q = q.detach().float().cpu().numpy() if isinstance(q, torch.Tensor) else np.asarray(q)
        q = np.ascontiguousarray(q, dtype=np.float32)
        if not np.all(np.isfinite(q)):
            raise ValueError("non-finite entries in queries")
        if q.ndim != 4:
            raise ValueError("queries must have shape (steps, layers, q_heads, dim)")
        if min(q.shape[1:]) < 1:
            raise ValueError(f"layer/head/dim axes must be positive, got {q.shape}")
        if self.gqa_group < 1:
            raise ValueError("gqa_group must be >= 1")
        if q.shape[2] % self.gqa_group != 0:
            raise ValueError(f"num_query_heads {q.shape[2]} not divisible by gqa_group {self.gqa_group}")
        object.__setattr__(self, "queries", q)

    @property
    def num_steps(self):
        return self.queries.shape[0]

    @property
    def num_layers(self):
        return self.queries.shape[1]

    @property
    def num_query_heads(self):
        return self.queries.shape[2]

    @property
    def head_dim(self):
        return self.queries.shape[3]

    def kv_head_for(self, query_head):
        return query_head // self.gqa_group

    def query(self, step, layer, query_head):
        """One float32 query vector of length head_dim."""
        return self.queries[step, layer, query_head]

    def step_queries(self, step, layer, device=None, dtype=torch.float32):
        """All q heads of one (step, layer) as a device tensor [1, Hq, d]."""
        t = torch.from_numpy(self.queries[step, layer]).unsqueeze(0)
        return t.to(device if device is not None else torch.device("cuda")).to(dtype)


@dataclass
class Cluster:
    """`clustering.py:110-118` (host copy of one device cluster)."""

    members: np.ndarray
    centroid: np.ndarray
    size: int
    value_mean: np.ndarray

    @property
    def value_sum(self):
        return self.value_mean * self.size


class EstimationData:
    """`clustering.py:121-127`: dense centroid / log-size / value-mean arrays
    plus the cluster list of one head, copied from the device tables (fp32
    centroids and value means, as stored for decode).  Also indexable by the
    ``head_tables`` keys ("members", "centroids", "value_means", "sizes",
    "offs")."""

    def __init__(self, tables):
        self._t = tables
        self.centroids = tables["centroids"]
        self.value_means = tables["value_means"]
        self.log_sizes = np.log(tables["sizes"].astype(np.float64))
        self.clusters = [Cluster(members=m, centroid=c, size=int(sz), value_mean=vm) for m, c, sz, vm in
                         zip(tables["members"], tables["centroids"], tables["sizes"], tables["value_means"])]

    def __getitem__(self, key):
        return self._t[key]


class ClusteredCache:
    """Per-layer clustered view of one sequence (`clustering.py:140-258`).
    ``source`` is the cache object the caller passed (identity-checked by
    sparse_attention / recovered_mass, as in the reference); ``device_source``
    its device copy."""

    def __init__(self, source, sink, window, layers, device_source=None):
        self.source, self.sink, self.window = source, sink, window
        self.device_source = device_source if device_source is not None else source
        self.layers = layers
        self._est = {}

    @property
    def num_appended(self):
        return self.layers[0].n_tokens - self.source.context_len

    @property
    def total_tokens(self):
        return self.layers[0].n_tokens

    @property
    def middle_range(self):
        return (self.sink, self.source.context_len - self.window)

    def sink_token_indices(self):
        return np.arange(self.sink, dtype=np.int64)

    def window_token_indices(self):
        t = self.total_tokens
        return np.arange(t - self.window, t, dtype=np.int64)

    def append_tokens(self, new_keys, new_values):
        """`clustering.py:182-196`: new_keys/new_values [L, Hkv, d]."""
        nk = torch.as_tensor(new_keys)
        nv = torch.as_tensor(new_values)
        want = (self.source.num_layers, self.source.num_kv_heads, self.source.head_dim)
        if tuple(nk.shape) != want or tuple(nv.shape) != want:
            raise ValueError(f"appended token must have shape {want}")
        if not (torch.isfinite(nk.float()).all() and torch.isfinite(nv.float()).all()):
            raise ValueError("non-finite entries in appended token")
        dev = self.layers[0].device
        for li, lay in enumerate(self.layers):
            lay.append(nk[li].unsqueeze(0).to(dev), nv[li].unsqueeze(0).to(dev))
        self._est.clear()

    def estimation_data(self, layer, kv_head):
        """`clustering.py:243-258`: host copy of one head's tables (cached
        until the next append)."""
        key = (layer, kv_head, self.total_tokens)
        hit = self._est.get(key)
        if hit is None:
            hit = self._est[key] = EstimationData(self.layers[layer].head_tables(0, kv_head))
        return hit

    def head_clusters(self, layer, kv_head):
        """`clustering.py:219-229`: middle clusters plus residual singletons."""
        return self.estimation_data(layer, kv_head).clusters

    @property
    def clusters(self):
        """`clusters[layer][kv_head]`: the prefill (middle-range) clusters."""
        stop = self.source.context_len - self.window
        return [[[c for c in self.head_clusters(li, h) if c.members[0] < stop]
                 for h in range(self.source.num_kv_heads)] for li in range(len(self.layers))]

    def _rows_of(self, layer, kv_head, positions):
        lay = self.layers[layer]
        positions = np.asarray(positions, dtype=np.int64)
        mid_end = lay.prefill_tokens - lay.window
        rows = positions.copy()
        inmid = (positions >= lay.sink) & (positions < mid_end)
        if inmid.any():
            perm = lay.perm[0, kv_head, :mid_end].cpu().numpy().astype(np.int64)
            inv = np.empty(mid_end, dtype=np.int64)
            inv[perm[lay.sink:mid_end]] = np.arange(lay.sink, mid_end)
            rows[inmid] = inv[positions[inmid]]
        return rows

    def gather_keys(self, layer, kv_head, positions):
        """`clustering.py:198-203`: host f32 key rows at token positions."""
        rows = torch.from_numpy(self._rows_of(layer, kv_head, positions)).to(self.layers[layer].device)
        lay = self.layers[layer]
        return lay.keys[0, kv_head, :, :lay.dim].index_select(0, rows).float().cpu().numpy()

    def gather_values(self, layer, kv_head, positions):
        rows = torch.from_numpy(self._rows_of(layer, kv_head, positions)).to(self.layers[layer].device)
        lay = self.layers[layer]
        return lay.values[0, kv_head, :, :lay.dim].index_select(0, rows).float().cpu().numpy()


# device clustered caches made from the reference's ClusteredCache objects
_DEV_CLUSTERED = {}


def device_clustered(cc, headroom=256):
    """This package's ClusteredCache for ``cc``: itself, or -- for the
    reference's ClusteredCache (clustering.py:140-258: host clusters from its
    own k-means) -- the same clusters uploaded into the device layout (sink
    rows, each cluster's members contiguous in cluster order, then the
    residual singletons and the window at their own positions; fp32
    centroids and value means).  Made once per object; tokens appended to
    the reference object since are appended here too."""
    if isinstance(cc, ClusteredCache):
        return cc
    if not (hasattr(cc, "clusters") and hasattr(cc, "source") and hasattr(cc, "head_clusters")):
        raise TypeError(f"expected a ClusteredCache, got {type(cc).__name__}")
    key = id(cc)
    hit = _DEV_CLUSTERED.get(key)
    if hit is not None and hit[0]() is cc:
        ours = hit[1]
        have, want = ours.num_appended, int(cc.num_appended)
        if have == want:
            return ours
        if have < want:
            for j in range(have, want):
                ours.append_tokens(cc._extra_keys[j], cc._extra_values[j])
            return ours
    ours = _upload_reference_clustered(cc, headroom)
    try:
        ref = weakref.ref(cc, lambda _r, k=key: _DEV_CLUSTERED.pop(k, None))
        _DEV_CLUSTERED[key] = (ref, ours)
    except TypeError:
        pass
    return ours


def _upload_reference_clustered(cc, headroom):
    src = cc.source
    L, H, n, d = (src.num_layers, src.num_kv_heads, src.context_len, src.head_dim)
    sink, window = int(cc.sink), int(cc.window)
    dev = torch.device("cuda")
    keys = np.asarray(src.keys, dtype=np.float32)
    values = np.asarray(src.values, dtype=np.float32)
    dl, d = d, ((d + 7) // 8) * 8  # device rows zero-padded to a multiple of 8
    if d != dl:
        keys = np.concatenate([keys, np.zeros(keys.shape[:3] + (d - dl,), np.float32)], 3)
        values = np.concatenate([values, np.zeros(values.shape[:3] + (d - dl,), np.float32)], 3)
    mid_end = n - window
    kmax = max(len(cc.clusters[li][h]) for li in range(L) for h in range(H))
    cap, row_cap = kmax + headroom, n + headroom
    layers = []
    for li in range(L):
        K = np.zeros((1, H, row_cap, d), np.float32)
        V = np.zeros_like(K)
        offs = np.zeros((1, H, cap + 1), np.int32)
        ncl = np.zeros((1, H), np.int32)
        cents = np.zeros((1, H, cap, d), np.float32)
        vbar = np.zeros_like(cents)
        perm = np.zeros((1, H, row_cap), np.int32)
        for h in range(H):
            cl = cc.clusters[li][h]
            order = np.concatenate([np.arange(sink)] + [np.asarray(c.members, np.int64) for c in cl] +
                                   [np.arange(mid_end, n)])
            if order.size != n:
                raise ValueError("clusters do not partition the middle token range")
            K[0, h, :n], V[0, h, :n] = keys[li, h, order], values[li, h, order]
            perm[0, h, :n] = order
            sizes = np.array([len(c.members) for c in cl], np.int64)
            offs[0, h, :len(cl) + 1] = sink + np.concatenate([[0], np.cumsum(sizes)])
            ncl[0, h] = len(cl)
            if cl:
                cents[0, h, :len(cl), :dl] = np.stack([np.asarray(c.centroid, np.float64) for c in cl])
                vbar[0, h, :len(cl), :dl] = np.stack([np.asarray(c.value_mean, np.float64) for c in cl])
        t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
        lay = ClusteredLayer(t(K), t(V), t(offs), t(ncl), t(cents), t(vbar), t(perm), n, sink, window,
                             prefill_tokens=n, logical_dim=dl)
        lay._prefill_k = kmax
        layers.append(lay)
    ours = ClusteredCache(src, sink, window, layers, device_source=device_cache(src))
    for j in range(int(cc.num_appended)):
        ours.append_tokens(cc._extra_keys[j], cc._extra_values[j])
    return ours


def build_clustered_cache(cache, k=None, sink=4, window=64, seed=0, max_iters=DEFAULT_MAX_ITERS,
                          tokens_per_cluster=DEFAULT_TOKENS_PER_CLUSTER, growth=0, fp64_assign=True):
    """`clustering.py:266-314` on the GPU.  ``cache`` is this package's
    KvCache or any object with [L, Hkv, N, d] ``keys``/``values`` (the
    reference's KvCache); the returned ClusteredCache keeps it as ``source``.
    ``growth`` pre-reserves rows/clusters for that many appended tokens
    (appends past it reallocate)."""
    dev = device_cache(cache)
    if isinstance(cache, (tuple, list)):
        cache = dev
    layers = []
    for li in range(dev.num_layers):
        layers.append(cluster_layer(
            dev.keys[li:li + 1], dev.values[li:li + 1], k=k, sink=sink, window=window, seed=seed,
            max_iters=max_iters, tokens_per_cluster=tokens_per_cluster, layer=li, fp64_assign=fp64_assign,
            row_cap=dev.context_len + growth, extra_clusters=growth))
        layers[-1].logical_dim = dev.head_dim
    return ClusteredCache(cache, sink, window, layers, device_source=dev)
