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
                 window, objective=None, iters=None, prefill_tokens=None):
        self.keys, self.values = keys, values
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
        want = (self.batch, self.kv_heads, self.head_dim)
        if tuple(new_k.shape) != want or tuple(new_v.shape) != want:
            raise ValueError(f"appended token must have shape {want}")
        if self.n_tokens >= self.row_cap:
            raise ValueError("row capacity exhausted")
        if self.n_tokens - self.window >= self.sink and \
                self.n_tokens - self.prefill_tokens + 1 > self.cluster_cap - self._prefill_k:
            raise ValueError("cluster table capacity exhausted")
        nk = new_k.to(self.dtype).contiguous()
        nv = new_v.to(self.dtype).contiguous()
        v = self.view()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        N.check(N.lib().dp_append_token(v, N.ptr(nk), N.ptr(nv), st.cuda_stream))
        self.n_tokens += 1
        self._keep = (nk, nv)

    _prefill_k = 0

    def split(self):
        """One single-sequence ClusteredLayer per batch entry, sharing storage
        (used to cluster many layers in one launch, then hand them out)."""
        out = []
        for b in range(self.batch):
            sl = lambda t: None if t is None else t[b:b + 1]  # noqa: E731
            lay = ClusteredLayer(sl(self.keys), sl(self.values), sl(self.offs), sl(self.nclusters),
                                 sl(self.centroids), sl(self.value_means), sl(self.perm), self.n_tokens,
                                 self.sink, self.window, prefill_tokens=self.prefill_tokens)
            lay._prefill_k = self._prefill_k
            out.append(lay)
        return out

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
            "centroids": self.centroids[b, h, :K].double().cpu().numpy(),
            "value_means": self.value_means[b, h, :K].double().cpu().numpy(),
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
# reference-signature containers (kvcache.py:50-139, clustering.py:140-314)
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
        object.__setattr__(self, "keys", k.to(dev).contiguous())
        object.__setattr__(self, "values", v.to(dev).contiguous())

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
        return self.keys.shape[3]


class ClusteredCache:
    """Per-layer clustered view of one sequence (`clustering.py:140-258`)."""

    def __init__(self, source, sink, window, layers):
        self.source, self.sink, self.window = source, sink, window
        self.layers = layers

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
        dev = self.layers[0].device
        for li, lay in enumerate(self.layers):
            lay.append(nk[li].unsqueeze(0).to(dev), nv[li].unsqueeze(0).to(dev))

    def estimation_data(self, layer, kv_head):
        """Host view of one head's tables (members, centroids, value means)."""
        return self.layers[layer].head_tables(0, kv_head)


def build_clustered_cache(cache, k=None, sink=4, window=64, seed=0, max_iters=DEFAULT_MAX_ITERS,
                          tokens_per_cluster=DEFAULT_TOKENS_PER_CLUSTER, growth=0, fp64_assign=True):
    """`clustering.py:266-314` on the GPU.  ``growth`` reserves rows/clusters
    for that many appended tokens."""
    if not isinstance(cache, KvCache):
        cache = KvCache(*cache)
    layers = []
    for li in range(cache.num_layers):
        layers.append(cluster_layer(
            cache.keys[li:li + 1], cache.values[li:li + 1], k=k, sink=sink, window=window, seed=seed,
            max_iters=max_iters, tokens_per_cluster=tokens_per_cluster, layer=li, fp64_assign=fp64_assign,
            row_cap=cache.context_len + growth, extra_clusters=growth))
    return ClusteredCache(cache, sink, window, layers)
