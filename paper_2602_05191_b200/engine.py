"""Double-P decode step on the GPU, behind the reference's operator API.

Reference: /root/reference/pkg/src/doublep/engine.py.  Two entry styles:

* product path (batched, device tensors, no host sync):
      out = sparse_attention(q, layer, p1=0.95, p2=0.7)        # q [B, Hq, d]
  where ``layer`` is a ``ClusteredLayer``; plus ``dense_attention`` (the
  full-attention comparator) and ``DecodeWorkspace`` to preallocate.

* reference signatures (per (layer, kv head), single query vector), for the
  parity suite and drop-in use:
      decode_step(q, cache, cc, cfg, layer, kv_head) -> (AttentionOutput,
          SelectionPlan, ClusterEstimate)
      estimate_cluster_distribution, plan_selection, sparse_attention(q,
      cache, cc, plan, layer, kv_head), full_attention (the token-level
      baselines and metrics.py quantities live in metrics.py)

Every result is computed by libdoublep_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .cache import (ClusteredCache, ClusteredLayer, KvCache, default_cluster_count, device_cache, device_clustered,
                    dtype_code, pad_dim)


@dataclass(frozen=True)
class DoublePConfig:
    """`engine.py:33-60`."""

    p1: float
    p2: float
    sink: int = 4
    window: int = 64
    clusters: int | None = None
    tokens_per_cluster: int = 32

    def __post_init__(self):
        for name, val in (("p1", self.p1), ("p2", self.p2)):
            if not 0.0 < val <= 1.0:
                raise ValueError(f"{name} must be in (0, 1], got {val}")
        if self.sink < 0 or self.window < 0:
            raise ValueError("sink and window must be >= 0")

    def cluster_count_for(self, middle_len):
        if self.clusters is not None:
            return self.clusters
        return default_cluster_count(middle_len, self.tokens_per_cluster)


PRESETS = {"llama-default": (0.95, 0.7), "qwen-default": (0.99, 0.8)}  # engine.py:64-67


class DecodeWorkspace:
    """All step buffers for one layer geometry and GQA group, allocated once
    (nothing allocates on the step path)."""

    def __init__(self, layer: ClusteredLayer, gqa_group: int):
        B, H, d, cap = layer.batch, layer.kv_heads, layer.head_dim, layer.cluster_cap
        dev = layer.device
        G = int(gqa_group)
        self.G, self.key = G, self._key(layer, G)
        self.log_mass = torch.zeros((B, H * G, cap), dtype=torch.float64, device=dev)
        self.state = torch.zeros((B, H * G, cap), dtype=torch.uint8, device=dev)
        self.counts = torch.zeros((B, H * G, 2), dtype=torch.int32, device=dev)
        self.out = torch.zeros((B, H * G, d), dtype=torch.float32, device=dev)
        self.lse = torch.zeros((B, H * G), dtype=torch.float32, device=dev)
        self.stats = torch.zeros((B, H, 4), dtype=torch.int32, device=dev)
        nbytes = N.lib().dp_decode_workspace_bytes(layer.view(), G)
        self.ws = torch.zeros((max(nbytes, 1),), dtype=torch.uint8, device=dev)  # counters start at 0

    @staticmethod
    def _key(layer, G):
        return (layer.batch, layer.kv_heads, layer.head_dim, layer.row_cap, layer.cluster_cap, G,
                str(layer.dtype))

    def fits(self, layer, G):
        return self.key == self._key(layer, G)


def _group(q, layer):
    if q.dim() != 3 or q.shape[0] != layer.batch or q.shape[2] != layer.head_dim:
        raise ValueError(f"dimension mismatch: query {tuple(q.shape)}, cache (B={layer.batch}, "
                         f"d={layer.head_dim})")
    if q.shape[1] % layer.kv_heads:
        raise ValueError(f"num_query_heads {q.shape[1]} not divisible by kv heads {layer.kv_heads}")
    return q.shape[1] // layer.kv_heads


def _stream(layer, stream):
    return (stream if stream is not None else torch.cuda.current_stream(layer.device)).cuda_stream


def sparse_attention(q, cache, *args, **kw):
    """Product path ``sparse_attention(q[B,Hq,d], layer, p1, p2, ...)`` or the
    reference signature ``sparse_attention(q, cache, cc, plan, layer,
    kv_head)`` (engine.py:255-264)."""
    if isinstance(cache, ClusteredLayer):
        return _sparse_layer(q, cache, *args, **kw)
    return _sparse_ref(q, cache, *args, **kw)


def _sparse_layer(q, layer, p1=0.95, p2=0.7, *, workspace=None, return_plan=False, stream=None,
                  scale=None, out=None):
    """One decode step over a whole layer: score -> two-stage top-p ->
    mixed exact/approx attention.  Returns out fp32 [B,Hq,d] (and the
    workspace holding log_mass/state/counts/lse/stats if return_plan).
    `out`, if given, is a contiguous fp32 CUDA tensor [B,Hq,d] written in
    place (lets one workspace serve every layer while outputs accumulate)."""
    for name, val in (("p1", p1), ("p2", p2)):
        if not 0.0 < val <= 1.0:
            raise ValueError(f"{name} must be in (0, 1], got {val}")
    G = _group(q, layer)
    ws = workspace if workspace is not None and workspace.fits(layer, G) else DecodeWorkspace(layer, G)
    if out is None:
        out = ws.out
    elif out.dtype != torch.float32 or tuple(out.shape) != tuple(ws.out.shape) or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous float32 tensor of shape {tuple(ws.out.shape)}")
    q = q.contiguous()
    sc = layer.attn_scale if scale is None else scale
    N.check(N.lib().dp_decode_step(
        layer.view(), N.ptr(q), dtype_code(q), G, sc, p1, p2, N.ptr(ws.log_mass), N.ptr(ws.state),
        N.ptr(ws.counts), N.ptr(out), N.ptr(ws.lse), N.ptr(ws.stats), N.ptr(ws.ws), ws.ws.numel(),
        _stream(layer, stream)))
    return (out, ws) if return_plan else out


class DecodeGraph:
    """One decode step over several layers captured as a CUDA graph -- the
    serving-engine form of the product path.  Every replay runs, for each
    layer li, exactly the eager ``sparse_attention(q[li], layers[li], p1, p2)``
    launches (plan + attend, PDL-chained) into ``out[li]``, without the
    per-call host work.  ``q`` [L,B,Hq,d] and ``out`` [L,B,Hq,d] fp32 are fixed
    device buffers.  Optional pinned host buffers move inside the graph:
    ``host_q`` is copied in (layer 0's slice first, the rest on a side stream
    while layer 0 runs) and the outputs are copied to ``host_out`` on a side
    stream every ``out_every`` layers, so only the last batch's copy is
    exposed.  Layers share one geometry (and one workspace, reused layer
    after layer as in the eager path).

    The captured launches hold each layer's token count, so a graph is valid
    for one cache state: after ``ClusteredLayer.append`` (decode-time growth)
    ``replay()`` raises -- rebuild the graph (or call ``recapture()``)."""

    def __init__(self, layers, q, p1=0.95, p2=0.7, *, out=None, workspace=None, host_q=None, host_out=None,
                 out_every=8):
        for name, val in (("p1", p1), ("p2", p2)):
            if not 0.0 < val <= 1.0:
                raise ValueError(f"{name} must be in (0, 1], got {val}")
        if q.dim() != 4 or q.shape[0] != len(layers):
            raise ValueError(f"q must be [layers, B, Hq, d] with {len(layers)} layers, got {tuple(q.shape)}")
        G = _group(q[0], layers[0])
        ws = workspace if workspace is not None else DecodeWorkspace(layers[0], G)
        for lay in layers:
            if not ws.fits(lay, G):
                raise ValueError("DecodeGraph layers must share one geometry (the workspace does not fit)")
        dev = layers[0].device
        self.layers, self.q, self.ws = list(layers), q, ws
        self.out = out if out is not None else torch.empty(q.shape, dtype=torch.float32, device=dev)
        if self.out.dtype != torch.float32 or self.out.shape != q.shape or not self.out.is_contiguous():
            raise ValueError(f"out must be a contiguous float32 tensor of shape {tuple(q.shape)}")
        for name, t, dt in (("host_q", host_q, q.dtype), ("host_out", host_out, torch.float32)):
            if t is not None and (t.shape != q.shape or t.dtype != dt or t.is_cuda or not t.is_pinned()):
                raise ValueError(f"{name} must be a pinned host tensor of shape {tuple(q.shape)} and dtype {dt}")
        self.host_q, self.host_out = host_q, host_out
        # layers per device->host output copy: every copy forks a side-stream
        # branch off the layer chain, which breaks the programmatic (PDL)
        # overlap of the next layer's launch, so copies are batched
        self.out_every = max(1, int(out_every))
        self.p1, self.p2 = p1, p2
        self._s_in, self._s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        self._step()  # eager warm-up (allocates nothing): caches attributes, tensor maps, views
        torch.cuda.synchronize(dev)
        self._capture()

    def _capture(self):
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._step()
        self._ntok = [lay.n_tokens for lay in self.layers]

    def recapture(self):
        """Re-record the graph for the layers' current token counts."""
        torch.cuda.synchronize(self.layers[0].device)
        self._capture()

    def _step(self):
        main = torch.cuda.current_stream(self.layers[0].device)
        hq, ho = self.host_q, self.host_out
        if hq is not None:
            self.q[0].copy_(hq[0], non_blocking=True)
            if len(self.layers) > 1:
                self._s_in.wait_stream(main)
                with torch.cuda.stream(self._s_in):
                    self.q[1:].copy_(hq[1:], non_blocking=True)
        for li, lay in enumerate(self.layers):
            if li == 1 and hq is not None:
                main.wait_stream(self._s_in)
            _sparse_layer(self.q[li], lay, self.p1, self.p2, workspace=self.ws, out=self.out[li])
            if ho is not None and ((li + 1) % self.out_every == 0 or li + 1 == len(self.layers)):
                l0 = (li // self.out_every) * self.out_every
                self._s_out.wait_stream(main)
                with torch.cuda.stream(self._s_out):
                    ho[l0:li + 1].copy_(self.out[l0:li + 1], non_blocking=True)
        if ho is not None:
            main.wait_stream(self._s_out)

    def replay(self):
        if [lay.n_tokens for lay in self.layers] != self._ntok:
            raise ValueError("DecodeGraph is stale: a layer's token count changed since capture "
                             "(append_tokens); call recapture()")
        self.graph.replay()
        return self.host_out if self.host_out is not None else self.out


def cluster_topk_attention(q, layer, budget, *, workspace=None, stream=None, scale=None, return_plan=False):
    """Fixed cluster-budget baseline on the device (baseline_cluster_topk,
    engine.py:318-338): the `budget` clusters of largest estimated mass are
    exact, every other cluster is approximated -- the RetroInfer-style
    comparator of PAPER.md:505.  Returns out fp32 [B,Hq,d] (and the
    workspace with log_mass/state/order/counts if return_plan)."""
    if int(budget) < 1:
        raise ValueError(f"cluster budget must be >= 1, got {budget}")
    G = _group(q, layer)
    ws = workspace if workspace is not None and workspace.fits(layer, G) else DecodeWorkspace(layer, G)
    if getattr(ws, "order", None) is None:
        ws.order = torch.zeros(ws.state.shape, dtype=torch.int32, device=ws.state.device)
    q = q.contiguous()
    sc = layer.attn_scale if scale is None else scale
    N.check(N.lib().dp_cluster_topk(
        layer.view(), N.ptr(q), dtype_code(q), G, sc, int(budget), N.ptr(ws.log_mass), N.ptr(ws.state),
        N.ptr(ws.order), N.ptr(ws.counts), N.ptr(ws.out), N.ptr(ws.lse), N.ptr(ws.stats), N.ptr(ws.ws),
        ws.ws.numel(), _stream(layer, stream)))
    return (ws.out, ws) if return_plan else ws.out


def dense_attention(q, layer, *, workspace=None, stream=None, scale=None, return_lse=False):
    """Dense split-KV flash decoding over every cached row (full_attention,
    engine.py:122-144) -- the comparator the sparse step must beat."""
    G = _group(q, layer)
    ws = workspace if workspace is not None and workspace.fits(layer, G) else DecodeWorkspace(layer, G)
    q = q.contiguous()
    sc = layer.attn_scale if scale is None else scale
    N.check(N.lib().dp_dense_attention(layer.view(), N.ptr(q), dtype_code(q), G, sc, N.ptr(ws.out),
                                       N.ptr(ws.lse), N.ptr(ws.ws), ws.ws.numel(), _stream(layer, stream)))
    return (ws.out, ws.lse) if return_lse else ws.out


# ---------------------------------------------------------------------------
# reference-signature API (engine.py:70-278)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TopPResult:
    """`selection.py:16-33`."""

    selected: np.ndarray
    cumulative_mass: float
    p: float


@dataclass(frozen=True)
class ClusterEstimate:
    """`engine.py:70-85`; ``_dev`` keeps the device log-masses."""

    log_masses: np.ndarray
    probs: np.ndarray
    order: np.ndarray
    cc: ClusteredCache
    layer: int
    kv_head: int
    _dev: object = None


@dataclass(frozen=True)
class SelectionPlan:
    """`engine.py:88-102`."""

    stage1: TopPResult
    exact_clusters: np.ndarray
    approx_clusters: np.ndarray
    exact_tokens: np.ndarray
    estimate: ClusterEstimate
    config: DoublePConfig
    _state: object = None


@dataclass(frozen=True)
class AttentionOutput:
    """`engine.py:105-112` (+ the log normaliser the kernels return)."""

    output: np.ndarray
    normalizer: float
    exact_token_count: int
    approx_cluster_count: int
    log_normalizer: float = 0.0


def _check_query(q, d):
    q = torch.as_tensor(q)
    if tuple(q.shape) != (d,):
        raise ValueError(f"dimension mismatch: query {tuple(q.shape)}, head_dim {d}")
    return q


def _head_q(q, lay):
    qt = torch.as_tensor(q, device=lay.device)
    if qt.dtype not in (torch.float32, torch.bfloat16):
        qt = qt.float()
    return pad_dim(qt.reshape(1, 1, -1), lay.head_dim).contiguous()


class _HeadBufs:
    def __init__(self, lay, dev):
        cap = lay.cluster_cap
        self.lm = torch.zeros((1, 1, cap), dtype=torch.float64, device=dev)
        self.state = torch.zeros((1, 1, cap), dtype=torch.uint8, device=dev)
        self.counts = torch.zeros((1, 1, 2), dtype=torch.int32, device=dev)
        self.order = torch.zeros((1, 1, cap), dtype=torch.int32, device=dev)
        self.probs = torch.zeros((1, 1, cap), dtype=torch.float64, device=dev)
        self.cum = torch.zeros((1, 1), dtype=torch.float64, device=dev)


def estimate_cluster_distribution(q, cc, layer, kv_head):
    """`engine.py:158-177` via dp_score (+ the softmax/order of dp_select).
    ``cc`` may also be the reference's ClusteredCache (uploaded once)."""
    cc = device_clustered(cc)
    lay = cc.layers[layer]
    K = int(lay.nclusters[0, kv_head].item())
    if K == 0:
        raise ValueError("no clusters for this head")
    _check_query(q, cc.source.head_dim)
    qd = _head_q(q, lay)
    bufs = _HeadBufs(lay, lay.device)
    v = lay.view(0, kv_head)
    st = torch.cuda.current_stream(lay.device).cuda_stream
    N.check(N.lib().dp_score(v, N.ptr(qd), dtype_code(qd), 1, lay.attn_scale,
                             N.ptr(bufs.lm), st))
    # stage thresholds irrelevant here; p=1 keeps the full order
    N.check(N.lib().dp_select(v, 1, 1.0, 1.0, N.ptr(bufs.lm), N.ptr(bufs.state), N.ptr(bufs.counts),
                              N.ptr(bufs.order), N.ptr(bufs.cum), N.ptr(bufs.probs), None, 0, st))
    return ClusterEstimate(
        log_masses=bufs.lm[0, 0, :K].cpu().numpy(), probs=bufs.probs[0, 0, :K].cpu().numpy(),
        order=bufs.order[0, 0, :K].cpu().numpy().astype(np.int64), cc=cc, layer=layer, kv_head=kv_head,
        _dev=(bufs, qd))


def plan_selection(est, cfg):
    """`engine.py:180-213` via dp_select."""
    cc, layer, h = est.cc, est.layer, est.kv_head
    lay = cc.layers[layer]
    bufs, qd = est._dev
    K = est.log_masses.size
    v = lay.view(0, h)
    st = torch.cuda.current_stream(lay.device).cuda_stream
    N.check(N.lib().dp_select(v, 1, cfg.p1, cfg.p2, N.ptr(bufs.lm), N.ptr(bufs.state), N.ptr(bufs.counts),
                              N.ptr(bufs.order), N.ptr(bufs.cum), N.ptr(bufs.probs), None, 0, st))
    n1, n2 = (int(x) for x in bufs.counts[0, 0].cpu())
    order = bufs.order[0, 0, :K].cpu().numpy().astype(np.int64)
    cp = order[:n1]
    tables = lay.head_tables(0, h)
    tokens = np.concatenate([cc.sink_token_indices(), cc.window_token_indices(),
                             *[tables["members"][int(i)] for i in cp[:n2]]])
    tokens.sort()
    return SelectionPlan(
        stage1=TopPResult(selected=cp, cumulative_mass=float(bufs.cum[0, 0].item()), p=cfg.p1),
        exact_clusters=cp[:n2], approx_clusters=cp[n2:], exact_tokens=tokens, estimate=est, config=cfg,
        _state=bufs.state.clone())


def _sparse_ref(q, cache, cc, plan, layer, kv_head):
    """`engine.py:255-264` via dp_sparse_attention on the plan's device state."""
    if cc.source is not cache:
        raise ValueError("plan/cc mismatch: clustered cache built from a different cache")
    cc = device_clustered(cc)
    est = plan.estimate
    if est.cc is not cc or est.layer != layer or est.kv_head != kv_head:
        raise ValueError("plan/cc mismatch: plan was derived for a different head or cache")
    lay = cc.layers[layer]
    _check_query(q, lay.dim)
    qd = _head_q(q, lay)
    bufs, _ = est._dev
    out = torch.zeros((1, 1, lay.head_dim), dtype=torch.float32, device=lay.device)
    lse = torch.zeros((1, 1), dtype=torch.float32, device=lay.device)
    v = lay.view(0, kv_head)
    ws = torch.zeros((N.lib().dp_decode_workspace_bytes(v, 1),), dtype=torch.uint8, device=lay.device)
    st = torch.cuda.current_stream(lay.device).cuda_stream
    N.check(N.lib().dp_sparse_attention(v, N.ptr(qd), dtype_code(qd), 1, lay.attn_scale,
                                        N.ptr(bufs.lm), N.ptr(plan._state), N.ptr(out), N.ptr(lse), None,
                                        N.ptr(ws), ws.numel(), st))
    lz = float(lse.item())
    return AttentionOutput(output=out[0, 0, :lay.dim].double().cpu().numpy(), normalizer=math.exp(lz),
                           exact_token_count=int(plan.exact_tokens.size),
                           approx_cluster_count=int(plan.approx_clusters.size), log_normalizer=lz)


def decode_step(q, cache, cc, cfg, layer, kv_head):
    """`engine.py:267-278`."""
    if cc.sink != cfg.sink or cc.window != cfg.window:
        raise ValueError(
            "config/cache mismatch: clustered cache was built with "
            f"sink={cc.sink}, window={cc.window}, config has sink={cfg.sink}, window={cfg.window}")
    cc = device_clustered(cc)
    est = estimate_cluster_distribution(q, cc, layer, kv_head)
    plan = plan_selection(est, cfg)
    out = _sparse_ref(q, cache, cc, plan, layer, kv_head)
    return out, plan, est


def full_attention(q, cache, layer, kv_head, cc=None):
    """Dense oracle signature (`engine.py:135-144`) on the GPU dense kernel.
    With ``cc`` it covers the grown token range (true_token_weights)."""
    if cc is not None:
        cc = device_clustered(cc)
    src = cache if cc is None else cc.source
    d = src.head_dim
    _check_query(q, d)
    if cc is not None:
        lay = cc.layers[layer]
        v = lay.view(0, kv_head)
        n = lay.n_tokens
        dev = lay.device
    else:
        dc = device_cache(cache)
        k = dc.keys[layer, kv_head].unsqueeze(0).unsqueeze(0).contiguous()
        vv = dc.values[layer, kv_head].unsqueeze(0).unsqueeze(0).contiguous()
        n = k.shape[2]
        dev = k.device
        dp_ = k.shape[3]
        dummy_i = torch.zeros((1, 1, 2), dtype=torch.int32, device=dev)
        dummy_f = torch.zeros((1, 1, 1, dp_), dtype=torch.float32, device=dev)
        lay = ClusteredLayer(k, vv, dummy_i, dummy_i[..., 0], dummy_f, dummy_f, None, n, 0, 0, logical_dim=d)
        v = lay.view()
    qd = _head_q(q, lay)
    out = torch.zeros((1, 1, lay.head_dim), dtype=torch.float32, device=dev)
    lse = torch.zeros((1, 1), dtype=torch.float32, device=dev)
    ws = torch.zeros((N.lib().dp_decode_workspace_bytes(v, 1),), dtype=torch.uint8, device=dev)
    N.check(N.lib().dp_dense_attention(v, N.ptr(qd), dtype_code(qd), 1, lay.attn_scale, N.ptr(out),
                                       N.ptr(lse), N.ptr(ws), ws.numel(),
                                       torch.cuda.current_stream(dev).cuda_stream))
    lz = float(lse.item())
    return AttentionOutput(output=out[0, 0, :d].double().cpu().numpy(), normalizer=math.exp(lz),
                           exact_token_count=n, approx_cluster_count=0, log_normalizer=lz)


def build_cache_for_config(cache, cfg, seed=0):
    """`engine.py:281-290`."""
    from .cache import build_clustered_cache

    middle = cache.context_len - cfg.sink - cfg.window
    k = cfg.cluster_count_for(middle) if hasattr(cfg, "cluster_count_for") else \
        (cfg.clusters if cfg.clusters is not None else default_cluster_count(middle, cfg.tokens_per_cluster))
    return build_clustered_cache(cache, k=k, sink=cfg.sink, window=cfg.window, seed=seed)
