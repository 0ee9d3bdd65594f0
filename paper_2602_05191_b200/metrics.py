"""Measurement side of the reference on the GPU.

Reference: /root/reference/pkg/src/doublep/metrics.py and the baselines in
engine.py:293-338.  Two entry styles, as in engine.py:

* batched device API over a whole ``ClusteredLayer`` (no host sync):
      w, lse = token_weights(q, layer)                         # true distribution
      out, captured, sel = token_topk_attention(q, layer, budget, weights=w)
      recovered_mass_batched(layer, w, state)                  # per q head
      cluster_approx_error_batched(layer, w, lse, log_mass, order)
      adaptive_token_budget_batched(layer, w, p)
      mixed_attention_f64(q, layer, state, log_mass)           # fp64 evaluation path
* reference signatures (per (layer, kv head), single query vector):
      recovered_mass(plan, q, cache), adaptive_token_budget(q, cache, p, layer,
      kv_head), violation_rate(recovered, p), cluster_approx_error(q, cache,
      cc, layer, kv_head), output_error(candidate, reference)

Everything is computed by libdoublep_b200.so (metrics.cu) in fp64, like the
reference; there is no CPU fallback.  Weights are in the layer's PHYSICAL
row order (cluster-contiguous); ``to_positions`` reorders them by token
position.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .cache import ClusteredLayer, device_cache, device_clustered, dtype_code
from .engine import AttentionOutput, _check_query, _group, _head_q, _stream, estimate_cluster_distribution


# ---------------------------------------------------------------------------
# batched device API
# ---------------------------------------------------------------------------


def token_weights(q, layer, *, scale=None, stream=None):
    """True attention distribution of every q head over all cached rows
    (full_attention_weights / true_token_weights, engine.py:122-155).
    Returns (weights fp64 [B,Hq,row_cap] physical row order, lse fp64 [B,Hq])."""
    G = _group(q, layer)
    q = q.contiguous()
    B, Hq = q.shape[0], q.shape[1]
    w = torch.zeros((B, Hq, layer.row_cap), dtype=torch.float64, device=layer.device)
    lse = torch.zeros((B, Hq), dtype=torch.float64, device=layer.device)
    sc = layer.attn_scale if scale is None else scale
    N.check(N.lib().dp_token_weights(layer.view(), N.ptr(q), dtype_code(q), G, sc, N.ptr(w), N.ptr(lse),
                                     _stream(layer, stream)))
    return w, lse


def _perm_args(layer):
    if layer.perm is None:
        return None, 0
    return N.ptr(layer.perm), layer.prefill_tokens - layer.window


def token_topk_attention(q, layer, budget, *, weights=None, budgets=None, scale=None, stream=None,
                         return_selected=False):
    """Idealised fixed-budget baseline (baseline_token_topk, engine.py:293-315)
    for every q head: the `budget` tokens of largest true weight (ties ->
    lower position), renormalised.  Returns (out fp64 [B,Hq,d], captured fp64
    [B,Hq]) and, with return_selected, the uint8 [B,Hq,row_cap] row mask.
    ``budgets`` (int32 [B,Hq], optional) caps each head's budget."""
    G = _group(q, layer)
    if not 1 <= int(budget) <= layer.n_tokens:
        raise ValueError(f"budget must be in [1, {layer.n_tokens}], got {budget}")
    if weights is None:
        weights, _ = token_weights(q, layer, scale=scale, stream=stream)
    B, Hq = q.shape[0], q.shape[1]
    out = torch.zeros((B, Hq, layer.head_dim), dtype=torch.float64, device=layer.device)
    cap = torch.zeros((B, Hq), dtype=torch.float64, device=layer.device)
    sel = torch.zeros((B, Hq, layer.row_cap), dtype=torch.uint8, device=layer.device) if return_selected else None
    perm, perm_rows = _perm_args(layer)
    N.check(N.lib().dp_token_topk(layer.view(), perm, perm_rows, G, int(budget), N.ptr(budgets), N.ptr(weights), N.ptr(out),
                                  N.ptr(cap), N.ptr(sel), _stream(layer, stream)))
    return (out, cap, sel) if return_selected else (out, cap)


def _g_of(layer, weights):
    Hq = weights.shape[1]
    if Hq % layer.kv_heads:
        raise ValueError(f"num_query_heads {Hq} not divisible by kv heads {layer.kv_heads}")
    return Hq // layer.kv_heads


def recovered_mass_batched(layer, weights, state, *, stream=None):
    """metrics.recovered_mass (metrics.py:26-39) per q head: true mass of
    sink + window + the state==2 clusters.  state uint8 [B,Hq,cluster_cap]."""
    G = _g_of(layer, weights)
    rec = torch.zeros(weights.shape[:2], dtype=torch.float64, device=layer.device)
    N.check(N.lib().dp_recovered_mass(layer.view(), G, N.ptr(weights), N.ptr(state.contiguous()), N.ptr(rec),
                                      _stream(layer, stream)))
    return rec


def cluster_approx_error_batched(layer, weights, lse, log_mass, order, *, stream=None):
    """metrics.cluster_approx_error (metrics.py:61-76) per q head, in
    estimated-rank order: errors fp64 [B,Hq,cluster_cap] (first K valid)."""
    G = _g_of(layer, weights)
    err = torch.zeros(log_mass.shape, dtype=torch.float64, device=layer.device)
    N.check(N.lib().dp_cluster_approx_error(layer.view(), G, N.ptr(weights), N.ptr(lse), N.ptr(log_mass),
                                            N.ptr(order), N.ptr(err), _stream(layer, stream)))
    return err


def adaptive_token_budget_batched(layer, weights, p, *, stream=None):
    """metrics.adaptive_token_budget (metrics.py:41-50) per q head: the
    minimal token count whose true mass reaches p.  int32 [B,Hq]."""
    G = _g_of(layer, weights)
    out = torch.zeros(weights.shape[:2], dtype=torch.int32, device=layer.device)
    N.check(N.lib().dp_adaptive_token_budget(layer.view(), G, N.ptr(weights), float(p), N.ptr(out),
                                             _stream(layer, stream)))
    return out


def mixed_attention_f64(q, layer, state=None, log_mass=None, *, scale=None, stream=None):
    """mixed_attention (engine.py:216-252) in fp64 for every q head with the
    plan given as per-cluster states (2 exact, 1 approx, 0 dropped); no state
    = every cluster exact, i.e. full attention.  Deterministic -- the
    experiment runner's evaluation path.  Returns (out fp64 [B,Hq,d], lse
    fp64 [B,Hq])."""
    G = _group(q, layer)
    q = q.contiguous()
    B, Hq = q.shape[0], q.shape[1]
    out = torch.zeros((B, Hq, layer.head_dim), dtype=torch.float64, device=layer.device)
    lse = torch.zeros((B, Hq), dtype=torch.float64, device=layer.device)
    sc = layer.attn_scale if scale is None else scale
    N.check(N.lib().dp_mixed_attention_f64(layer.view(), N.ptr(q), dtype_code(q), G, sc, N.ptr(log_mass),
                                           N.ptr(None if state is None else state.contiguous()), N.ptr(out),
                                           N.ptr(lse), _stream(layer, stream)))
    return out, lse


def to_positions(layer, rows, b=0, h=0):
    """Reorder a [..., row_cap] per-row tensor of head (b, h) by token
    position (host numpy, first n_tokens entries)."""
    x = rows[..., :layer.n_tokens].cpu().numpy()
    if layer.perm is None:
        return x
    pos = np.arange(layer.n_tokens)
    mid_end = layer.prefill_tokens - layer.window
    pos[:mid_end] = layer.perm[b, h, :mid_end].cpu().numpy()
    outp = np.empty_like(x)
    outp[..., pos] = x
    return outp


# ---------------------------------------------------------------------------
# reference signatures (metrics.py / engine.py)
# ---------------------------------------------------------------------------


def output_error(candidate, reference):
    """Relative L2 error (metrics.py:15-23)."""
    a = candidate.output if hasattr(candidate, "output") else np.asarray(candidate)
    b = reference.output if hasattr(reference, "output") else np.asarray(reference)
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    return float(np.linalg.norm(a - b)) / max(float(np.linalg.norm(b)), 1e-12)


def _dense_head_layer(cache, layer, kv_head):
    """A one-head ClusteredLayer over a plain KvCache (no tables); ``cache``
    may be the reference's numpy KvCache (copied to the device once)."""
    dc = device_cache(cache)
    k = dc.keys[layer, kv_head].unsqueeze(0).unsqueeze(0).contiguous()
    v = dc.values[layer, kv_head].unsqueeze(0).unsqueeze(0).contiguous()
    d = k.shape[-1]
    di = torch.zeros((1, 1, 2), dtype=torch.int32, device=k.device)
    df = torch.zeros((1, 1, 1, d), dtype=torch.float32, device=k.device)
    return ClusteredLayer(k, v, di, di[..., 0], df, df, None, k.shape[2], 0, 0, logical_dim=dc.head_dim)


def _head_weights(q, lay, kv_head):
    """(weights [1,1,row_cap] device, lse float) of one q vector on head kv_head."""
    qd = _head_q(q, lay)
    v = lay.view(0, kv_head)
    w = torch.zeros((1, 1, lay.row_cap), dtype=torch.float64, device=lay.device)
    lse = torch.zeros((1, 1), dtype=torch.float64, device=lay.device)
    N.check(N.lib().dp_token_weights(v, N.ptr(qd), dtype_code(qd), 1, lay.attn_scale, N.ptr(w),
                                     N.ptr(lse), torch.cuda.current_stream(lay.device).cuda_stream))
    return v, w, lse


def full_attention_weights(q, cache, layer, kv_head):
    """engine.py:122-132: (weights f64[N] by position, lse)."""
    lay = _dense_head_layer(cache, layer, kv_head)
    _check_query(q, lay.dim)
    _, w, lse = _head_weights(q, lay, 0)
    return w[0, 0, :lay.n_tokens].cpu().numpy(), float(lse.item())


def true_token_weights(q, cc, layer, kv_head):
    """engine.py:147-155: like full_attention_weights over the grown range."""
    cc = device_clustered(cc)
    lay = cc.layers[layer]
    _check_query(q, lay.dim)
    _, w, lse = _head_weights(q, lay, kv_head)
    return to_positions(lay, w[0, 0], 0, kv_head), float(lse.item())


def baseline_token_topk(q, cache, budget, layer, kv_head):
    """engine.py:293-315: (AttentionOutput, captured)."""
    lay = _dense_head_layer(cache, layer, kv_head)
    _check_query(q, lay.dim)
    if not 1 <= budget <= lay.n_tokens:
        raise ValueError(f"budget must be in [1, {lay.n_tokens}], got {budget}")
    v, w, lse = _head_weights(q, lay, 0)
    out = torch.zeros((1, 1, lay.head_dim), dtype=torch.float64, device=lay.device)
    cap = torch.zeros((1, 1), dtype=torch.float64, device=lay.device)
    N.check(N.lib().dp_token_topk(v, None, 0, 1, int(budget), None, N.ptr(w), N.ptr(out), N.ptr(cap), None,
                                  torch.cuda.current_stream(lay.device).cuda_stream))
    captured = float(cap.item())
    lz = float(lse.item())
    return AttentionOutput(output=out[0, 0, :lay.dim].cpu().numpy(), normalizer=math.exp(lz) * captured,
                           exact_token_count=int(budget), approx_cluster_count=0,
                           log_normalizer=lz + math.log(captured)), captured


def recovered_mass(plan, q, cache):
    """metrics.py:26-39: true mass carried by a plan's exact tokens."""
    est = plan.estimate
    cc = est.cc
    if cc.source is not cache:
        raise ValueError("plan/cc mismatch: plan was derived from a different cache")
    lay = cc.layers[est.layer]
    _check_query(q, lay.dim)
    v, w, _ = _head_weights(q, lay, est.kv_head)
    rec = torch.zeros((1, 1), dtype=torch.float64, device=lay.device)
    N.check(N.lib().dp_recovered_mass(v, 1, N.ptr(w), N.ptr(plan._state), N.ptr(rec),
                                      torch.cuda.current_stream(lay.device).cuda_stream))
    return float(rec.item())


def adaptive_token_budget(q, cache, p, layer, kv_head):
    """metrics.py:41-50: minimal number of tokens whose true mass reaches p."""
    lay = _dense_head_layer(cache, layer, kv_head)
    _check_query(q, lay.dim)
    v, w, _ = _head_weights(q, lay, 0)
    out = torch.zeros((1, 1), dtype=torch.int32, device=lay.device)
    N.check(N.lib().dp_adaptive_token_budget(v, 1, N.ptr(w), float(p), N.ptr(out),
                                             torch.cuda.current_stream(lay.device).cuda_stream))
    return int(out.item())


def violation_rate(recovered, p):
    """metrics.py:53-58: fraction of steps whose recovered mass is below p."""
    arr = np.asarray(recovered, dtype=np.float64)
    if arr.size == 0:
        raise ValueError("no recovered masses given")
    return float(np.mean(arr < p))


def cluster_approx_error(q, cache, cc, layer, kv_head):
    """metrics.py:61-76: (errors in estimated-rank order, order)."""
    cc = device_clustered(cc)
    est = estimate_cluster_distribution(q, cc, layer, kv_head)
    lay = cc.layers[layer]
    bufs, _ = est._dev
    v, w, lse = _head_weights(q, lay, kv_head)
    err = torch.zeros(bufs.lm.shape, dtype=torch.float64, device=lay.device)
    N.check(N.lib().dp_cluster_approx_error(v, 1, N.ptr(w), N.ptr(lse), N.ptr(bufs.lm), N.ptr(bufs.order),
                                            N.ptr(err), torch.cuda.current_stream(lay.device).cuda_stream))
    K = est.order.size
    return err[0, 0, :K].cpu().numpy(), est.order


def baseline_cluster_topk(q, cache, cc, budget, layer, kv_head):
    """engine.py:318-338: the `budget` clusters of largest estimated mass
    exact, every other cluster approximated, sink and window exact (shared
    normaliser).  Device selection (dp_cluster_topk), fp64 evaluation."""
    from .engine import cluster_topk_attention

    cc = device_clustered(cc)
    est = estimate_cluster_distribution(q, cc, layer, kv_head)
    total = est.probs.size
    if not 1 <= budget <= total:
        raise ValueError(f"cluster budget must be in [1, {total}], got {budget}")
    hl = cc.layers[layer].head(0, kv_head)
    qd = _head_q(q, hl)
    _, ws = cluster_topk_attention(qd, hl, int(budget), return_plan=True)
    st = ws.state.clone()
    out, lse = mixed_attention_f64(qd, hl, st, ws.log_mass)
    stn = st[0, 0, :total].cpu().numpy()
    sizes = cc.estimation_data(layer, kv_head)["sizes"]
    exact = cc.sink + cc.window + int(sizes[stn == 2].sum())
    lz = float(lse[0, 0].item())
    return AttentionOutput(output=out[0, 0, :hl.dim].cpu().numpy(), normalizer=math.exp(lz), exact_token_count=exact,
                           approx_cluster_count=int((stn == 1).sum()), log_normalizer=lz)


def baseline_token_topp_fixed_budget(q, cache, est_budget, p, layer, kv_head):
    """engine.py:340-370: candidates = the top `est_budget` tokens of the true
    distribution, kept = the shortest candidate prefix whose true mass reaches
    p (all of them if it never does).  Returns (AttentionOutput over the kept
    tokens, renormalised; recovered true mass)."""
    lay = _dense_head_layer(cache, layer, kv_head)
    _check_query(q, lay.dim)
    if not 1 <= est_budget <= lay.n_tokens:
        raise ValueError(f"est_budget must be in [1, {lay.n_tokens}], got {est_budget}")
    qd = _head_q(q, lay)
    w, lse = token_weights(qd, lay)
    budgets = adaptive_token_budget_batched(lay, w, float(p))
    out, cap = token_topk_attention(qd, lay, int(est_budget), weights=w, budgets=budgets)
    kept = min(int(budgets[0, 0].item()), int(est_budget))
    rec = float(cap[0, 0].item())
    lz = float(lse[0, 0].item())
    return AttentionOutput(output=out[0, 0, :lay.dim].cpu().numpy(), normalizer=math.exp(lz) * rec, exact_token_count=kept,
                           approx_cluster_count=0, log_normalizer=lz + math.log(rec)), rec
