"""Experiment runner on the GPU: the ``b200`` backend of the reference CLI
(reference cli.py:1-717).

    python -m paper_2602_05191_b200.cli run   --n 4096 --d 128 --method doublep --steps 8
    python -m paper_2602_05191_b200.cli sweep --input w.dpkv --methods doublep,token_topk \
        --p1-grid 0.9,0.95,0.99 --k-grid 256,1024
    python -m paper_2602_05191_b200.cli gen | cluster | figs ...

Same subcommands, flags, methods, CSV/JSON schema and formatting as the
reference (CSV_COLUMNS cli.py:39-43, record fields metrics.py ExperimentRecord,
sweep aggregates cli.py:245-277, 12-significant-digit floats, atomic output
files, rows in (layer, head, step) order, one-line ``doublep: error:`` on
failure).  What differs is where the numbers come from:

* every quantity is computed on the GPU through libdoublep_b200.so, batched
  over all q heads of a (layer, step): clustering (dp_cluster_build),
  scoring/selection (dp_score, dp_select, dp_cluster_topk), the outputs in fp64
  (dp_mixed_attention_f64 / dp_token_topk -- deterministic, so repeated runs
  are byte-identical), the dense reference, recovered mass and budgets
  (metrics.cu);
* ``--input`` reads the reference's DPKV files (so a reference-generated
  workload gives the same inputs); inline workloads use the device
  generator of workload.py (the reference law, torch Philox streams), so they
  are deterministic but not the reference's NumPy draws;
* cluster tables hold fp32 centroids/value means (the decode layout), so
  float columns agree with the reference to ~1e-6 relative, not to 12 digits;
  integer columns (selection counts, exact tokens) agree exactly up to score
  ties (tests/test_gpu_cli.py).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys
import tempfile
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .cache import ClusteredLayer, cluster_layer, dtype_code
from .engine import PRESETS, cluster_topk_attention
from . import metrics as M

METHODS = ("full", "doublep", "token_topk", "cluster_topk", "token_topp_fixed")
PROFILES = ("peaked", "heavy", "uniform", "mixed")

CSV_COLUMNS = [
    "layer", "head", "step", "method", "p1", "p2", "k", "m", "B",
    "clusters_total", "clusters_selected", "clusters_exact", "exact_tokens",
    "est_mass", "recovered_mass", "violation", "rel_err",
]
SWEEP_COLUMNS = [
    "method", "p1", "p2", "k", "m", "B", "records",
    "mean_rel_err", "p50_rel_err", "p90_rel_err",
    "mean_exact_tokens", "violation_rate",
]


# ---------------------------------------------------------------------------
# configuration and records (reference workload.py:35-75, cli.py:46-72,
# metrics.py ExperimentRecord)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class WorkloadSpec:
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
            raise ValueError(f"tail_profile must be one of {PROFILES}, got {self.tail_profile!r}")
        for name in ("context_len", "head_dim", "num_layers", "num_kv_heads", "gqa_group", "num_steps",
                     "num_blobs"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.blob_spread < 0 or self.blob_separation <= 0:
            raise ValueError("blob_spread must be >= 0 and blob_separation > 0")
        if self.sink < 0 or self.window < 0:
            raise ValueError("sink and window must be >= 0")
        if self.context_len <= self.sink + self.window:
            raise ValueError(f"context_len {self.context_len} must exceed sink + window "
                             f"({self.sink} + {self.window})")


@dataclass(frozen=True)
class RunConfig:
    """One method run over one workload (cli.py:46-72)."""

    workload: WorkloadSpec | None
    input_path: str | None
    method: str
    p1: float = 0.95
    p2: float = 0.7
    k: int | None = None
    m: int | None = None
    B: int | None = None
    target_p: float = 0.95
    clusters: int | None = None
    tokens_per_cluster: int = 32
    sink: int = 4
    window: int = 64
    seed: int = 0

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}, expected one of {METHODS}")
        if (self.workload is None) == (self.input_path is None):
            raise ValueError("exactly one of workload or input_path must be given")


@dataclass(frozen=True)
class ExperimentRecord:
    """One (layer, head, step, method) row (metrics.py ExperimentRecord)."""

    layer: int
    head: int
    step: int
    method: str
    p1: float | None
    p2: float | None
    k: int | None
    m: int | None
    B: int | None
    clusters_total: int | None
    clusters_selected: int | None
    clusters_exact: int | None
    exact_tokens: int
    est_mass: float | None
    recovered_mass: float
    violation: bool
    rel_err: float

    def __post_init__(self):
        if not -1e-6 <= self.recovered_mass <= 1.0 + 1e-6:
            raise ValueError(f"recovered_mass out of range: {self.recovered_mass}")
        if self.rel_err < 0:
            raise ValueError(f"rel_err must be >= 0, got {self.rel_err}")


def _round12(x):
    return float(f"{x:.12g}")


# ---------------------------------------------------------------------------
# workloads on the device
# ---------------------------------------------------------------------------


class _Workload:
    """keys/values: one [1,H,N,d] fp32 CUDA tensor per layer; queries fp32
    numpy [S,L,Hq,d]."""

    def __init__(self, keys, values, queries):
        self.keys, self.values, self.queries = keys, values, np.ascontiguousarray(queries, dtype=np.float32)
        self.num_layers = len(keys)
        self.num_kv_heads, self.context_len, self.head_dim = keys[0].shape[1:]
        self.num_steps, _, self.num_query_heads, _ = self.queries.shape
        if self.num_query_heads % self.num_kv_heads:
            raise ValueError(f"num_query_heads {self.num_query_heads} not divisible by kv heads "
                             f"{self.num_kv_heads}")
        self.gqa_group = self.num_query_heads // self.num_kv_heads


def generate(spec, device="cuda"):
    """Device workload with the reference generator law (workload.py here)."""
    from .workload import generate_layer, generate_queries

    keys, values = [], []
    qs = np.zeros((spec.num_steps, spec.num_layers, spec.num_kv_heads * spec.gqa_group, spec.head_dim),
                  dtype=np.float32)
    for li in range(spec.num_layers):
        k, v, centers = generate_layer(1, spec.num_kv_heads, spec.context_len, spec.head_dim, layer=li,
                                       seed=spec.seed, num_blobs=spec.num_blobs, blob_spread=spec.blob_spread,
                                       blob_separation=spec.blob_separation, dtype=torch.float32, device=device)
        keys.append(k)
        values.append(v)
        qs[:, li] = generate_queries(centers, spec.gqa_group, spec.num_steps, profile=spec.tail_profile, layer=li,
                                     seed=spec.seed, num_blobs=spec.num_blobs)[:, 0]
    return _Workload(keys, values, qs)


def _load(config_or_path, spec=None):
    from .dpkv import load_dpkv

    path = config_or_path if isinstance(config_or_path, str) else config_or_path.input_path
    if path is not None:
        _, keys, values, q = load_dpkv(path, dtype=torch.float32)
        return _Workload(keys, values, np.array(q))
    return generate(spec if spec is not None else config_or_path.workload)


def _plain_layer(kd, vd, window_all=True):
    """Unclustered layer over position-ordered rows; window = n makes every
    row an exact row of dp_mixed_attention_f64 (dense attention)."""
    n, d = kd.shape[2], kd.shape[3]
    di = torch.zeros((1, kd.shape[1], 2), dtype=torch.int32, device=kd.device)
    df = torch.zeros((1, kd.shape[1], 1, d), dtype=torch.float32, device=kd.device)
    return ClusteredLayer(kd, vd, di, di[..., 0], df, df, None, n, 0, n if window_all else 0)


def _rel_err(out, full):
    num = (out - full).norm(dim=-1)
    den = full.norm(dim=-1).clamp_min(1e-12)
    return (num / den).cpu().numpy()


def _cluster(wl, config, li):
    return cluster_layer(wl.keys[li], wl.values[li], k=config.clusters, sink=config.sink, window=config.window,
                         seed=config.seed, tokens_per_cluster=config.tokens_per_cluster, layer=li)


def _sizes(lay):
    """Per-kv-head cluster sizes (host) and counts."""
    K = lay.nclusters[0].cpu().numpy()
    offs = lay.offs[0].cpu().numpy()
    return K, [np.diff(offs[h, :K[h] + 1]) for h in range(K.size)]


def _select(lay, q, G, p1, p2):
    """dp_score + dp_select (the reference's estimate + plan_selection) for
    every q head: (log_mass, state, counts, cum) device tensors."""
    H, cap = lay.kv_heads, lay.cluster_cap
    dev = lay.device
    lm = torch.zeros((1, H * G, cap), dtype=torch.float64, device=dev)
    st = torch.zeros((1, H * G, cap), dtype=torch.uint8, device=dev)
    cnt = torch.zeros((1, H * G, 2), dtype=torch.int32, device=dev)
    cum = torch.zeros((1, H * G), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    v = lay.view()
    N.check(N.lib().dp_score(v, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(lm), s))
    N.check(N.lib().dp_select(v, G, p1, p2, N.ptr(lm), N.ptr(st), N.ptr(cnt), None, N.ptr(cum), None, None, 0, s))
    return lm, st, cnt, cum


# ---------------------------------------------------------------------------
# run / sweep (cli.py:93-277)
# ---------------------------------------------------------------------------


def run(config):
    """One method over every (layer, query head, step); ExperimentRecord rows
    in (layer, head, step) order.  rel_err is against fp64 dense attention
    computed for every record."""
    if config.method == "token_topk" and config.k is None:
        raise ValueError("method token_topk requires k")
    if config.method == "cluster_topk" and config.m is None:
        raise ValueError("method cluster_topk requires m")
    if config.method == "token_topp_fixed" and config.B is None:
        raise ValueError("method token_topp_fixed requires B")
    wl = _load(config)
    G, Hq, n = wl.gqa_group, wl.num_query_heads, wl.context_len
    rows = {}
    for li in range(wl.num_layers):
        plain = _plain_layer(wl.keys[li], wl.values[li])
        token = _plain_layer(wl.keys[li], wl.values[li], window_all=False)
        lay = _cluster(wl, config, li) if config.method in ("doublep", "cluster_topk") else None
        if lay is not None:
            K, sizes = _sizes(lay)
        for step in range(wl.num_steps):
            q = torch.from_numpy(wl.queries[step, li].copy()).to(plain.device).unsqueeze(0)
            full, _ = M.mixed_attention_f64(q, plain)
            per = _step(config, q, full, plain, token, lay, G, n, K if lay is not None else None,
                        sizes if lay is not None else None)
            for head in range(Hq):
                rows[li, head, step] = ExperimentRecord(layer=li, head=head, step=step, method=config.method,
                                                        **per[head])
    return [rows[key] for key in sorted(rows)]


def _step(config, q, full, plain, token, lay, G, n, K, sizes):
    Hq = q.shape[1]
    none = dict(p1=None, p2=None, k=None, m=None, B=None, clusters_total=None, clusters_selected=None,
                clusters_exact=None, est_mass=None)
    tp = config.target_p
    if config.method == "full":
        return [dict(none, exact_tokens=n, recovered_mass=1.0, violation=bool(1.0 < tp), rel_err=0.0)
                for _ in range(Hq)]
    if config.method == "doublep":
        lm, st, cnt, cum = _select(lay, q, G, config.p1, config.p2)
        out, _ = M.mixed_attention_f64(q, lay, st, lm)
        w, _ = M.token_weights(q, lay)
        rec = M.recovered_mass_batched(lay, w, st).cpu().numpy()[0]
        err = _rel_err(out, full)[0]
        stn, cn, cu = st[0].cpu().numpy(), cnt[0].cpu().numpy(), cum[0].cpu().numpy()
        res = []
        for hq in range(Hq):
            h = hq // G
            exact = lay.sink + lay.window + int(sizes[h][stn[hq, :K[h]] == 2].sum())
            res.append(dict(none, p1=config.p1, p2=config.p2, clusters_total=int(K[h]),
                            clusters_selected=int(cn[hq, 0]), clusters_exact=int(cn[hq, 1]), exact_tokens=exact,
                            est_mass=_round12(float(cu[hq])), recovered_mass=_round12(float(rec[hq])),
                            violation=bool(rec[hq] < tp), rel_err=_round12(float(err[hq]))))
        return res
    if config.method == "cluster_topk":
        m = int(config.m)
        for h in range(K.size):
            if not 1 <= m <= int(K[h]):
                raise ValueError(f"cluster budget must be in [1, {int(K[h])}], got {m}")
        _, ws = cluster_topk_attention(q, lay, m, return_plan=True)
        st = ws.state.clone()
        out, _ = M.mixed_attention_f64(q, lay, st, ws.log_mass)
        w, _ = M.token_weights(q, lay)
        rec = M.recovered_mass_batched(lay, w, st).cpu().numpy()[0]
        err = _rel_err(out, full)[0]
        stn = st[0].cpu().numpy()
        res = []
        for hq in range(Hq):
            h = hq // G
            exact = lay.sink + lay.window + int(sizes[h][stn[hq, :K[h]] == 2].sum())
            res.append(dict(none, m=m, clusters_total=int(K[h]), clusters_selected=int(K[h]), clusters_exact=m,
                            exact_tokens=exact, recovered_mass=_round12(float(rec[hq])),
                            violation=bool(rec[hq] < tp), rel_err=_round12(float(err[hq]))))
        return res
    w, _ = M.token_weights(q, token)
    if config.method == "token_topk":
        out, cap = M.token_topk_attention(q, token, int(config.k), weights=w)
        err = _rel_err(out, full)[0]
        cap = cap.cpu().numpy()[0]
        return [dict(none, k=int(config.k), exact_tokens=int(config.k), recovered_mass=_round12(float(cap[hq])),
                     violation=bool(cap[hq] < tp), rel_err=_round12(float(err[hq]))) for hq in range(Hq)]
    # token_topp_fixed (engine.py:340-370)
    Bc = int(config.B)
    if not 1 <= Bc <= n:
        raise ValueError(f"est_budget must be in [1, {n}], got {Bc}")
    if not 0.0 < tp <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {tp}")
    budgets = M.adaptive_token_budget_batched(token, w, tp)
    out, cap = M.token_topk_attention(q, token, Bc, weights=w, budgets=budgets)
    kept = torch.clamp(budgets, max=Bc).cpu().numpy()[0]
    err = _rel_err(out, full)[0]
    cap = cap.cpu().numpy()[0]
    return [dict(none, B=Bc, exact_tokens=int(kept[hq]), recovered_mass=_round12(float(cap[hq])),
                 violation=bool(cap[hq] < tp), rel_err=_round12(float(err[hq]))) for hq in range(Hq)]


def sweep(configs):
    """Run several configurations; one aggregate row each (cli.py:245-277)."""
    if not configs:
        raise ValueError("sweep needs at least one configuration")
    out = []
    for config in configs:
        records = run(config)
        errs = np.array([r.rel_err for r in records])
        rec = np.array([r.recovered_mass for r in records], dtype=np.float64)
        out.append({
            "method": config.method,
            "p1": config.p1 if config.method == "doublep" else None,
            "p2": config.p2 if config.method == "doublep" else None,
            "k": config.k, "m": config.m, "B": config.B,
            "records": len(records),
            "mean_rel_err": _round12(errs.mean()),
            "p50_rel_err": _round12(float(np.percentile(errs, 50))),
            "p90_rel_err": _round12(float(np.percentile(errs, 90))),
            "mean_exact_tokens": _round12(float(np.mean([r.exact_tokens for r in records]))),
            "violation_rate": _round12(M.violation_rate(rec, configs[0].target_p)),
        })
    return out


# ---------------------------------------------------------------------------
# analysis tables (cli.py:490-610)
# ---------------------------------------------------------------------------


def _figs_budgets(args, wl):
    ks = [int(x) for x in args.k_list.split(",") if x]
    rows = {}
    for li in range(wl.num_layers):
        token = _plain_layer(wl.keys[li], wl.values[li], window_all=False)
        for step in range(wl.num_steps):
            q = torch.from_numpy(wl.queries[step, li].copy()).to(token.device).unsqueeze(0)
            w, _ = M.token_weights(q, token)
            caps = [M.token_topk_attention(q, token, k, weights=w)[1].cpu().numpy()[0] for k in ks]
            budget = M.adaptive_token_budget_batched(token, w, args.target_p)
            bud = budget.cpu().numpy()[0]
            if int(bud.max()) > wl.context_len:
                raise ValueError(f"budget must be in [1, {wl.context_len}], got {int(bud.max())}")
            acap = M.token_topk_attention(q, token, wl.context_len, weights=w, budgets=budget)[1].cpu().numpy()[0]
            for head in range(wl.num_query_heads):
                r = [{"layer": li, "head": head, "step": step, "selector": f"top{k}", "budget": k,
                      "captured": _round12(float(c[head])), "violation": bool(c[head] < args.target_p)}
                     for k, c in zip(ks, caps)]
                r.append({"layer": li, "head": head, "step": step, "selector": "adaptive", "budget": int(bud[head]),
                          "captured": _round12(float(acap[head])), "violation": bool(acap[head] < args.target_p)})
                rows[li, head, step] = r
    return [x for key in sorted(rows) for x in rows[key]], \
        ["layer", "head", "step", "selector", "budget", "captured", "violation"]


def _figs_recovery(args, wl):
    Bc = args.B or wl.context_len // 4
    rows = {}
    for li in range(wl.num_layers):
        token = _plain_layer(wl.keys[li], wl.values[li], window_all=False)
        for step in range(wl.num_steps):
            q = torch.from_numpy(wl.queries[step, li].copy()).to(token.device).unsqueeze(0)
            w, _ = M.token_weights(q, token)
            budgets = M.adaptive_token_budget_batched(token, w, args.target_p)
            cap = M.token_topk_attention(q, token, Bc, weights=w, budgets=budgets)[1].cpu().numpy()[0]
            for head in range(wl.num_query_heads):
                rows[li, head, step] = {"layer": li, "head": head, "step": step, "B": Bc,
                                        "recovered": _round12(float(cap[head])),
                                        "violation": bool(cap[head] < args.target_p)}
    return [rows[k] for k in sorted(rows)], ["layer", "head", "step", "B", "recovered", "violation"]


def _figs_cluster_error(args, wl, cfg):
    rows = []
    G = wl.gqa_group
    for li in range(wl.num_layers):
        lay = _cluster(wl, cfg, li)
        K, _ = _sizes(lay)
        per = []
        for step in range(wl.num_steps):
            q = torch.from_numpy(wl.queries[step, li].copy()).to(lay.device).unsqueeze(0)
            lm, _, _, _ = _select(lay, q, G, 1.0, 1.0)
            order = torch.zeros(lm.shape, dtype=torch.int32, device=lay.device)
            st, cnt = torch.zeros(lm.shape, dtype=torch.uint8, device=lay.device), \
                torch.zeros((1, lm.shape[1], 2), dtype=torch.int32, device=lay.device)
            N.check(N.lib().dp_select(lay.view(), G, 1.0, 1.0, N.ptr(lm), N.ptr(st), N.ptr(cnt), N.ptr(order), None,
                                      None, None, 0, torch.cuda.current_stream(lay.device).cuda_stream))
            w, lse = M.token_weights(q, lay)
            per.append(M.cluster_approx_error_batched(lay, w, lse, lm, order)[0].cpu().numpy())
        stacked = np.stack(per)  # [S, Hq, cap]
        for h in range(wl.num_kv_heads):
            e = stacked[:, h * G, :K[h]]  # the first q head of each kv head (cli.py:556)
            for rank in range(e.shape[1]):
                rows.append({"layer": li, "kv_head": h, "rank": rank,
                             "mean_error": _round12(float(e[:, rank].mean())),
                             "max_error": _round12(float(e[:, rank].max()))})
    return rows, ["layer", "kv_head", "rank", "mean_error", "max_error"]


def _figs_tracking(args, wl, cfg, p1, p2):
    """Chosen exact-cluster counts against the minimal counts needed
    (metrics.min_clusters_for_error, metrics.py:79-104): every candidate
    count is one fp64 mixed-attention launch over all q heads."""
    rows = {}
    G = wl.gqa_group
    for li in range(wl.num_layers):
        lay = _cluster(wl, cfg, li)
        plain = _plain_layer(wl.keys[li], wl.values[li])
        K, _ = _sizes(lay)
        for step in range(wl.num_steps):
            q = torch.from_numpy(wl.queries[step, li].copy()).to(lay.device).unsqueeze(0)
            full, _ = M.mixed_attention_f64(q, plain)
            lm, st, cnt, _ = _select(lay, q, G, p1, p2)
            out, _ = M.mixed_attention_f64(q, lay, st, lm)
            err = _rel_err(out, full)[0]
            order = torch.zeros(lm.shape, dtype=torch.int32, device=lay.device)
            st1, c1 = torch.zeros_like(st), torch.zeros_like(cnt)
            N.check(N.lib().dp_select(lay.view(), G, 1.0, 1.0, N.ptr(lm), N.ptr(st1), N.ptr(c1), N.ptr(order),
                                      None, None, None, 0, torch.cuda.current_stream(lay.device).cuda_stream))
            order = order[0].cpu().numpy()
            rank = np.full((wl.num_query_heads, lay.cluster_cap), -1)
            for hq in range(wl.num_query_heads):
                k = int(K[hq // G])
                rank[hq, order[hq, :k]] = np.arange(k)
            eps = np.full(err.shape, args.epsilon) if args.epsilon else np.maximum(err, 1e-12)
            needed = np.full(err.shape, -1)
            for count in range(int(K.max()) + 1):
                stc = np.where(rank < 0, 0, np.where(rank < count, 2, 1)).astype(np.uint8)
                oc, _ = M.mixed_attention_f64(q, lay, torch.from_numpy(stc).to(lay.device).unsqueeze(0), lm)
                ec = _rel_err(oc, full)[0]
                hit = (needed < 0) & (ec <= eps) & (count <= np.repeat(K, G))
                needed[hit] = count
                if (needed >= 0).all():
                    break
            cn = cnt[0].cpu().numpy()
            for head in range(wl.num_query_heads):
                att = bool(needed[head] >= 0)
                nd = int(needed[head]) if att else int(K[head // G])
                rows[li, head, step] = {"layer": li, "head": head, "step": step, "rel_err": _round12(float(err[head])),
                                        "clusters_exact": int(cn[head, 1]), "min_clusters": nd, "attained": att,
                                        "ratio": _round12(int(cn[head, 1]) / max(nd, 1))}
    return [rows[k] for k in sorted(rows)], ["layer", "head", "step", "rel_err", "clusters_exact", "min_clusters",
                                             "attained", "ratio"]


# ---------------------------------------------------------------------------
# output (cli.py:280-330)
# ---------------------------------------------------------------------------


def _cell(value):
    if value is None:
        return ""
    if isinstance(value, (bool, np.bool_)):
        return "1" if value else "0"
    if isinstance(value, float):
        return f"{value:.12g}"
    return str(value)


def render(rows, columns, fmt):
    if fmt == "json":
        return json.dumps([{c: r[c] for c in columns} for r in rows], indent=2) + "\n"
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(columns)
    for r in rows:
        w.writerow([_cell(r[c]) for c in columns])
    return buf.getvalue()


def emit(text, out_path):
    """stdout, or an atomic replace of out_path (no partial files)."""
    if out_path is None:
        sys.stdout.write(text)
        return
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(os.path.abspath(out_path)), prefix=".tmp-", suffix=".out")
    try:
        with os.fdopen(fd, "w") as fh:
            fh.write(text)
        os.replace(tmp, out_path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def record_row(r):
    return {c: getattr(r, c) for c in CSV_COLUMNS}


# ---------------------------------------------------------------------------
# argument parsing (cli.py:290-717)
# ---------------------------------------------------------------------------


def _workload_flags(p):
    p.add_argument("--n", type=int, help="context length")
    p.add_argument("--d", type=int, help="head dimension")
    p.add_argument("--layers", type=int, default=1)
    p.add_argument("--kv-heads", type=int, default=1)
    p.add_argument("--gqa-group", type=int, default=1)
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--blobs", type=int, default=8)
    p.add_argument("--spread", type=float, default=0.3)
    p.add_argument("--separation", type=float, default=1.0)
    p.add_argument("--profile", choices=PROFILES, default="mixed")


def _cluster_flags(p):
    p.add_argument("--clusters", type=int, help="fixed cluster count per head")
    p.add_argument("--tokens-per-cluster", type=int, default=32)
    p.add_argument("--sink", type=int, default=4)
    p.add_argument("--window", type=int, default=64)


def _threshold_flags(p):
    p.add_argument("--p1", type=float)
    p.add_argument("--p2", type=float)
    p.add_argument("--preset", choices=sorted(PRESETS), help="named (p1, p2) pair")


def _output_flags(p):
    p.add_argument("--format", choices=("csv", "json"), default="csv")
    p.add_argument("--out", help="output path (default: stdout)")


def _thresholds(args):
    p1, p2 = PRESETS[args.preset] if args.preset else (0.95, 0.7)
    return (args.p1 if args.p1 is not None else p1), (args.p2 if args.p2 is not None else p2)


def _spec(args):
    if args.n is None or args.d is None:
        raise ValueError("--n and --d are required unless --input is given")
    return WorkloadSpec(context_len=args.n, head_dim=args.d, num_layers=args.layers, num_kv_heads=args.kv_heads,
                        gqa_group=args.gqa_group, num_steps=args.steps, num_blobs=args.blobs,
                        blob_spread=args.spread, blob_separation=args.separation, tail_profile=args.profile,
                        seed=args.seed, sink=getattr(args, "sink", 4), window=getattr(args, "window", 64))


def _source(args):
    return (None, args.input) if args.input is not None else (_spec(args), None)


def _config(args, **over):
    workload, path = _source(args)
    p1, p2 = _thresholds(args)
    base = dict(workload=workload, input_path=path, method=getattr(args, "method", None), p1=p1, p2=p2,
                k=getattr(args, "k", None), m=getattr(args, "m", None), B=getattr(args, "B", None),
                target_p=args.target_p, clusters=args.clusters, tokens_per_cluster=args.tokens_per_cluster,
                sink=args.sink, window=args.window, seed=args.seed)
    base.update(over)
    return RunConfig(**base)


def _cmd_gen(args):
    from .dpkv import write_dpkv

    wl = generate(_spec(args))
    keys = torch.cat(wl.keys).cpu().numpy()
    values = torch.cat(wl.values).cpu().numpy()
    write_dpkv(args.out, keys, values, wl.queries)
    return 0


def _cmd_cluster(args):
    wl = _load(args.input, None if args.input is not None else _spec(args))
    cfg = RunConfig(workload=None, input_path="-", method="full", clusters=args.clusters,
                    tokens_per_cluster=args.tokens_per_cluster, sink=args.sink, window=args.window, seed=args.seed)
    report = {"context_len": wl.context_len, "head_dim": wl.head_dim, "sink": args.sink, "window": args.window,
              "heads": []}
    for li in range(wl.num_layers):
        K, sizes = _sizes(_cluster(wl, cfg, li))
        for h in range(wl.num_kv_heads):
            s = sizes[h]
            report["heads"].append({"layer": li, "kv_head": h, "clusters": int(K[h]), "min_size": int(s.min()),
                                    "mean_size": _round12(float(s.mean())), "max_size": int(s.max())})
    emit(json.dumps(report, indent=2) + "\n", args.out)
    return 0


def _cmd_run(args):
    records = run(_config(args))
    emit(render([record_row(r) for r in records], CSV_COLUMNS, args.format), args.out)
    return 0


def _grid(text, cast):
    return [cast(x) for x in text.split(",") if x]


def _cmd_sweep(args):
    p1, p2 = _thresholds(args)
    grids = {
        "doublep": [dict(p1=a, p2=b) for a in (_grid(args.p1_grid, float) if args.p1_grid else [p1])
                    for b in (_grid(args.p2_grid, float) if args.p2_grid else [p2])],
        "token_topk": [dict(k=k) for k in (_grid(args.k_grid, int) if args.k_grid else [None])],
        "cluster_topk": [dict(m=m) for m in (_grid(args.m_grid, int) if args.m_grid else [None])],
        "token_topp_fixed": [dict(B=b) for b in (_grid(args.B_grid, int) if args.B_grid else [None])],
    }
    configs = []
    for method in args.methods.split(","):
        for over in grids.get(method, [{}]):
            kw = dict(method=method, k=None, m=None, B=None)
            if method != "doublep":
                kw.update(p1=0.95, p2=0.7)  # RunConfig defaults, as the reference's sweep leaves them
            kw.update(over)
            configs.append(_config(args, **kw))
    emit(render(sweep(configs), SWEEP_COLUMNS, args.format), args.out)
    return 0


def _cmd_figs(args):
    wl = _load(args.input, None if args.input is not None else _spec(args))
    p1, p2 = _thresholds(args)
    cfg = RunConfig(workload=None, input_path="-", method="full", clusters=args.clusters,
                    tokens_per_cluster=args.tokens_per_cluster, sink=args.sink, window=args.window, seed=args.seed)
    if args.table == "budgets":
        rows, cols = _figs_budgets(args, wl)
    elif args.table == "recovery":
        rows, cols = _figs_recovery(args, wl)
    elif args.table == "cluster-error":
        rows, cols = _figs_cluster_error(args, wl, cfg)
    else:
        rows, cols = _figs_tracking(args, wl, cfg, p1, p2)
    emit(render(rows, cols, args.format), args.out)
    return 0


def build_parser():
    parser = argparse.ArgumentParser(prog="doublep", description="hierarchical top-p sparse attention experiments "
                                                                 "(B200 backend)")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("gen", help="synthesize a workload dump")
    _workload_flags(p)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p.set_defaults(func=_cmd_gen)

    p = sub.add_parser("cluster", help="cluster a workload, report stats")
    p.add_argument("--input", help="dump file path")
    _workload_flags(p)
    _cluster_flags(p)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out")
    p.set_defaults(func=_cmd_cluster)

    p = sub.add_parser("run", help="run one method, emit per-step records")
    p.add_argument("--input", help="dump file path")
    _workload_flags(p)
    _cluster_flags(p)
    _threshold_flags(p)
    p.add_argument("--method", choices=METHODS, required=True)
    p.add_argument("--k", type=int, help="token budget for token_topk")
    p.add_argument("--m", type=int, help="cluster budget for cluster_topk")
    p.add_argument("--B", type=int, help="candidate budget for token_topp_fixed")
    p.add_argument("--target-p", type=float, default=0.95)
    p.add_argument("--seed", type=int, default=0)
    _output_flags(p)
    p.set_defaults(func=_cmd_run)

    p = sub.add_parser("sweep", help="run a parameter grid, emit aggregates")
    p.add_argument("--input", help="dump file path")
    _workload_flags(p)
    _cluster_flags(p)
    _threshold_flags(p)
    p.add_argument("--methods", default="doublep", help="comma-separated method list")
    for g in ("p1", "p2", "k", "m", "B"):
        p.add_argument(f"--{g}-grid", help=f"comma-separated {g} values")
    p.add_argument("--target-p", type=float, default=0.95)
    p.add_argument("--seed", type=int, default=0)
    _output_flags(p)
    p.set_defaults(func=_cmd_sweep)

    p = sub.add_parser("figs", help="recompute standard analysis tables")
    p.add_argument("--table", choices=("budgets", "recovery", "cluster-error", "tracking"), required=True)
    p.add_argument("--input", help="dump file path")
    _workload_flags(p)
    _cluster_flags(p)
    _threshold_flags(p)
    p.add_argument("--k-list", default="64,256,1024")
    p.add_argument("--B", type=int, help="candidate budget (default n/4)")
    p.add_argument("--epsilon", type=float, help="error bound for tracking")
    p.add_argument("--target-p", type=float, default=0.95)
    p.add_argument("--seed", type=int, default=0)
    _output_flags(p)
    p.set_defaults(func=_cmd_figs)
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except Exception as exc:  # one-line diagnostic, nonzero exit
        print(f"doublep: error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
