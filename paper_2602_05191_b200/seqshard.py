"""Sequence-sharded Double-P with the reference's GLOBAL semantics (config 5,
>= 512K tokens over P GPUs; verdict item 7).

Each rank holds the contiguous token positions ``seq_shard_bounds(N, P, r)``
of every (sequence, kv head) at prefill.  The result must equal what the
reference computes on the WHOLE sequence, so:

* **Prefill clustering is global** (`shard_cluster_layer`).  k-means++
  (clustering.py:36-55) runs over all ranks' middle points: per centre, each
  rank folds the newest centre into its local squared distances and sums
  them (dp_kmpp_shard_dsq), the P sums are all-gathered, the rank holding the
  point where the GLOBAL running sum first exceeds u * total writes it
  (dp_kmpp_shard_pick) and an all-reduce hands the centre to every rank.
  Lloyd (clustering.py:58-107) assigns local points (dp_nearest_centroid,
  fp64), sums them per cluster in position order (dp_lloyd_shard_sums) and
  all-reduces the [K, d + 1] sums and counts; empty clusters are dropped with
  the ascending remap on every rank alike, and the loop stops when nothing
  was dropped and no assignment changed anywhere.  The random stream is the
  reference's, replayed on every rank.
* **The clustered cache is partitioned by cluster.**  Rank r owns a
  contiguous range of the global cluster ids (balanced by member count) with
  ALL of their members (ascending positions, clustering.py:301), so its
  local ClusteredLayer is one slice of the global table: log|C| is the
  global size and each approximated cluster's pseudo-row lives on exactly
  one rank.  Rank 0 also holds the sink rows, rank P - 1 the window.
* **Each decode step selects globally** (`seqshard_decode`).  Every rank
  scores its slice (dp_score), the per-rank log-mass slices are all-gathered
  into the global table, the two-stage top-p runs on it (dp_select_global;
  deterministic, so every rank derives the same plan), each rank attends
  over its own exact clusters and approximated pseudo-rows
  (dp_sparse_attention) and ONE all-gather of the partial (out, lse) plus
  the log-sum-exp merge kernel (dp_lse_merge) combines them.

Collectives run on ``torch.distributed`` (NCCL over NVLink on a box; gloo
in the tests, where two ranks share one GPU).  The row redistribution of the
prefill is an all-gather of the members (an all-to-all at scale); the
per-step traffic is Hq * K * 8 bytes of log-masses and Hq * (d + 1) * 4
bytes of partials per rank.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .cache import ClusteredLayer, _check_geometry, dtype_code, head_seed, rng_stream
from .sharding import seq_shard_bounds

DEFAULT_MAX_ITERS = 25


class Comm:
    """The collectives this module needs, over a torch.distributed group.
    With gloo the tensors travel through host memory (gloo's CUDA support is
    partial); with NCCL they stay on the device."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host = dist.get_backend(group) != "nccl"

    def _in(self, t):
        return t.cpu() if self.host else t

    def all_gather(self, t):
        """[world, *t.shape] stacked in rank order."""
        src = self._in(t.contiguous())
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        return torch.stack(parts).to(t.device)

    def all_reduce(self, t, op=dist.ReduceOp.SUM):
        """In place (returns t)."""
        src = self._in(t)
        dist.all_reduce(src, op=op, group=self.group)
        if src is not t:
            t.copy_(src)
        return t


@dataclass
class ShardInfo:
    """Where this rank's slice sits in the global tables, per (sequence, kv head)."""
    world: int
    rank: int
    n_tokens: int               # global context length
    sink: int
    window: int
    k_global: np.ndarray        # [B, H] global cluster count (after drops)
    c_lo: np.ndarray            # [world + 1, B, H] cluster-id boundaries of the ranks
    centroids: torch.Tensor     # [B, H, cap_g, d] fp64 global centroids (parity / reporting)
    value_means: torch.Tensor   # [B, H, cap_g, d] fp64
    sizes: torch.Tensor         # [B, H, cap_g] int64 global cluster sizes
    assignment: list            # per unit: int64 [middle] global assignment (position order)
    objective: list             # per unit: list of per-iteration objectives
    picks: list                 # per unit: int64 [k] k-means++ picks (global middle indices)


def _nearest(points, centroids, assign, sqdist):
    N.check(N.lib().dp_nearest_centroid(N.ptr(points), dtype_code(points), points.shape[0], points.shape[1],
                                        N.ptr(centroids), centroids.shape[0], 1, N.ptr(assign), N.ptr(sqdist),
                                        torch.cuda.current_stream(points.device).cuda_stream))


def _sums(points, assign, k, dev):
    """Local fp64 sums [k, d] and counts [k] of one unit's points per cluster."""
    n, d = points.shape
    sums = torch.zeros((k, d), dtype=torch.float64, device=dev)
    cnt = torch.zeros((k,), dtype=torch.int64, device=dev)
    wsb = N.lib().dp_lloyd_shard_workspace_bytes(1, n, k)
    ws = torch.empty((max(wsb, 1),), dtype=torch.uint8, device=dev)
    N.check(N.lib().dp_lloyd_shard_sums(N.ptr(points), dtype_code(points), 1, n, d, N.ptr(assign), k, N.ptr(sums),
                                        N.ptr(cnt), N.ptr(ws), ws.numel(),
                                        torch.cuda.current_stream(dev).cuda_stream))
    return sums, cnt


def _kmeans_unit(comm, pts, gbase, middle, k, seed, max_iters):
    """Global k-means of one (sequence, kv head) unit over the ranks' local
    points `pts` [n_r, d] (global middle indices [gbase, gbase + n_r))."""
    dev = pts.device
    n, d = pts.shape
    st = torch.cuda.current_stream(dev).cuda_stream
    lib = N.lib()
    first, us, _alts = rng_stream(seed, middle, k)
    centres = torch.zeros((k, d), dtype=torch.float64, device=dev)
    cbuf = torch.zeros((1, d), dtype=torch.float64, device=dev)
    pick = torch.zeros((1,), dtype=torch.int32, device=dev)
    picks = np.zeros(k, dtype=np.int64)
    dsq = torch.zeros((1, n), dtype=torch.float64, device=dev)
    sums = torch.zeros((1,), dtype=torch.float64, device=dev)
    udraw = torch.from_numpy(np.asarray(us, dtype=np.float64)).to(dev)
    pin = torch.tensor([int(first)], dtype=torch.int32, device=dev)
    # ---- k-means++ (clustering.py:36-55)
    for i in range(k):
        if i == 0:
            N.check(lib.dp_kmpp_shard_pick(N.ptr(pts), dtype_code(pts), 1, n, d, None, None, comm.world, comm.rank,
                                           None, N.ptr(pin), gbase, N.ptr(cbuf), N.ptr(pick), st))
        else:
            allsums = comm.all_gather(sums)  # [P, 1]
            N.check(lib.dp_kmpp_shard_pick(N.ptr(pts), dtype_code(pts), 1, n, d, N.ptr(dsq), N.ptr(allsums),
                                           comm.world, comm.rank, N.ptr(udraw[i - 1:i]), None, gbase, N.ptr(cbuf),
                                           N.ptr(pick), st))
        got = comm.all_gather(pick.to(torch.int64))  # [P, 1]: the owner's global index, -1 elsewhere
        g = int(got.max().item())
        if g < 0:
            raise NotImplementedError("degenerate k-means++ seeding (all points coincide with centres) "
                                      "is not supported on the sequence-sharded path")
        picks[i] = g
        comm.all_reduce(cbuf)
        centres[i] = cbuf[0]
        if i + 1 < k:
            N.check(lib.dp_kmpp_shard_dsq(N.ptr(pts), dtype_code(pts), 1, n, d, N.ptr(centres[i:i + 1]),
                                          1 if i == 0 else 0, N.ptr(dsq), N.ptr(sums), st))
    # ---- Lloyd (clustering.py:58-107)
    assign = torch.zeros((n,), dtype=torch.int32, device=dev)
    sqd = torch.zeros((n,), dtype=torch.float64, device=dev)
    prev = None
    objective = []
    for _ in range(max_iters):
        kc = centres.shape[0]
        _nearest(pts, centres.contiguous(), assign, sqd)
        obj = comm.all_reduce(sqd.sum().reshape(1))
        objective.append(float(obj.item()))
        cnt = torch.bincount(assign.long(), minlength=kc)[:kc]
        comm.all_reduce(cnt)
        used = cnt > 0
        dropped = bool((~used).any().item())
        if dropped:
            remap = torch.cumsum(used.to(torch.int64), 0) - 1
            assign = remap[assign.long()].to(torch.int32)
            centres = centres[used]
        changed = torch.zeros((1,), dtype=torch.int64, device=dev)
        if prev is not None and not dropped:
            changed[0] = (assign != prev).sum()
        comm.all_reduce(changed)
        if not dropped and prev is not None and int(changed.item()) == 0:
            break
        prev = assign.clone()
        s, c = _sums(pts, assign, centres.shape[0], dev)
        comm.all_reduce(s)
        comm.all_reduce(c)
        centres = s / c.clamp(min=1).to(torch.float64).unsqueeze(1)
    s, c = _sums(pts, assign, centres.shape[0], dev)  # final exact means (clustering.py:104-106)
    comm.all_reduce(s)
    comm.all_reduce(c)
    centres = s / c.clamp(min=1).to(torch.float64).unsqueeze(1)
    return centres, c, assign, objective, picks


def _balanced_bounds(sizes, world):
    """Cluster-id boundaries [world + 1] giving every rank ~1/world of the members."""
    cum = np.concatenate([[0], np.cumsum(sizes)])
    total = cum[-1]
    b = [0]
    for r in range(1, world):
        b.append(int(np.searchsorted(cum, total * r / world, side="left")))
    b.append(len(sizes))
    return np.maximum.accumulate(np.asarray(b, dtype=np.int64))


def shard_cluster_layer(keys, values, n_tokens, comm: Comm, *, k=None, sink=4, window=64, seed=0,
                        max_iters=DEFAULT_MAX_ITERS, tokens_per_cluster=32, layer=0):
    """Global clustering of one layer from this rank's token slice.

    keys/values: CUDA [B, H, hi - lo, d] (f32 or bf16), the positions
    ``seq_shard_bounds(n_tokens, world, rank)`` of the sequence.  Returns
    (ClusteredLayer of this rank's cluster slice, ShardInfo)."""
    B, H, nl, d = keys.shape
    P, r = comm.world, comm.rank
    lo, hi = seq_shard_bounds(n_tokens, P, r)
    if nl != hi - lo:
        raise ValueError(f"rank {r} holds {nl} tokens, expected [{lo}, {hi}) of {n_tokens}")
    k, middle = _check_geometry(n_tokens, sink, window, k, tokens_per_cluster)
    m_lo, m_hi = max(lo, sink), min(hi, n_tokens - window)  # my middle positions
    if m_hi <= m_lo:
        raise ValueError("every rank must hold middle tokens (shard the sequence over fewer ranks)")
    gbase = m_lo - sink
    dev = keys.device
    U = B * H
    kk = keys.contiguous().reshape(U, nl, d)
    vv = values.contiguous().reshape(U, nl, d)
    results = []
    for u in range(U):
        b, h = divmod(u, H)
        pts = kk[u, m_lo - lo:m_hi - lo].contiguous()
        cents, cnt, assign, obj, picks = _kmeans_unit(comm, pts, gbase, middle, k, head_seed(seed, layer, h, b),
                                                      max_iters)
        vs, vc = _sums(vv[u, m_lo - lo:m_hi - lo].contiguous(), assign, cents.shape[0], dev)
        comm.all_reduce(vs)
        vbar = vs / cnt.clamp(min=1).to(torch.float64).unsqueeze(1)
        results.append((cents, cnt, assign, obj, picks, vbar))
    # ---- global assignment + rows of every rank (an all-to-all at scale)
    nmax_local = torch.tensor([m_hi - m_lo], dtype=torch.int64, device=dev)
    nmax = int(comm.all_reduce(nmax_local.clone(), op=dist.ReduceOp.MAX).item())
    kmax = int(comm.all_reduce(torch.tensor([max(x[0].shape[0] for x in results)], dtype=torch.int64, device=dev),
                               op=dist.ReduceOp.MAX).item())
    c_lo = np.zeros((P + 1, B, H), dtype=np.int64)
    k_glob = np.zeros((B, H), dtype=np.int64)
    per_unit = []
    for u in range(U):
        b, h = divmod(u, H)
        cents, cnt, assign, obj, picks, vbar = results[u]
        kc = cents.shape[0]
        k_glob[b, h] = kc
        sizes = cnt.cpu().numpy()
        c_lo[:, b, h] = _balanced_bounds(sizes, P)
        # gather every rank's (position, assignment, key, value) of this unit
        n_my = m_hi - m_lo
        pos = torch.full((nmax,), -1, dtype=torch.int64, device=dev)
        pos[:n_my] = torch.arange(m_lo, m_hi, device=dev)
        asg = torch.full((nmax,), -1, dtype=torch.int64, device=dev)
        asg[:n_my] = assign.long()
        kr = torch.zeros((nmax, d), dtype=keys.dtype, device=dev)
        vr = torch.zeros((nmax, d), dtype=keys.dtype, device=dev)
        kr[:n_my] = kk[u, m_lo - lo:m_hi - lo]
        vr[:n_my] = vv[u, m_lo - lo:m_hi - lo]
        all_pos = comm.all_gather(pos).reshape(-1)
        all_asg = comm.all_gather(asg).reshape(-1)
        all_k = comm.all_gather(kr).reshape(-1, d)
        all_v = comm.all_gather(vr).reshape(-1, d)
        ok = all_pos >= 0
        all_pos, all_asg, all_k, all_v = all_pos[ok], all_asg[ok], all_k[ok], all_v[ok]
        order = torch.argsort(all_pos)
        all_pos, all_asg, all_k, all_v = all_pos[order], all_asg[order], all_k[order], all_v[order]
        c0, c1 = int(c_lo[r, b, h]), int(c_lo[r + 1, b, h])
        mine = (all_asg >= c0) & (all_asg < c1)
        # members of my clusters: by cluster, ascending position inside each (stable sort)
        srt = torch.sort(all_asg[mine], stable=True)
        rows_pos = all_pos[mine][srt.indices]
        rows_k = all_k[mine][srt.indices]
        rows_v = all_v[mine][srt.indices]
        counts = torch.bincount(srt.values - c0, minlength=c1 - c0)[:c1 - c0]
        per_unit.append(dict(kc=kc, c0=c0, c1=c1, rows_pos=rows_pos, rows_k=rows_k, rows_v=rows_v, counts=counts,
                             cents=cents, vbar=vbar, glob_assign=all_asg, cnt=cnt, obj=obj, picks=picks))
    # ---- this rank's ClusteredLayer (one slice of the global table)
    my_sink = sink if r == 0 else 0
    my_window = window if r == P - 1 else 0
    max_rows = max(int(x["rows_pos"].numel()) for x in per_unit)
    cap = max(1, int(comm.all_reduce(torch.tensor([max(x["c1"] - x["c0"] for x in per_unit)], dtype=torch.int64,
                                                  device=dev), op=dist.ReduceOp.MAX).item()))
    n_loc = my_sink + max_rows + my_window
    dk = torch.zeros((B, H, n_loc, d), dtype=keys.dtype, device=dev)
    dv = torch.zeros_like(dk)
    offs = torch.zeros((B, H, cap + 1), dtype=torch.int32, device=dev)
    ncl = torch.zeros((B, H), dtype=torch.int32, device=dev)
    cents32 = torch.zeros((B, H, cap, d), dtype=torch.float32, device=dev)
    vbar32 = torch.zeros_like(cents32)
    perm = torch.full((B, H, n_loc), -1, dtype=torch.int32, device=dev)
    capg = kmax
    gc = torch.zeros((B, H, capg, d), dtype=torch.float64, device=dev)
    gv = torch.zeros_like(gc)
    gs = torch.zeros((B, H, capg), dtype=torch.int64, device=dev)
    assignments, objectives, picks_all = [], [], []
    for u in range(U):
        b, h = divmod(u, H)
        x = per_unit[u]
        kc, c0, c1 = x["kc"], x["c0"], x["c1"]
        nr = int(x["rows_pos"].numel())
        if my_sink:
            dk[b, h, :my_sink] = kk[u, :my_sink]
            dv[b, h, :my_sink] = vv[u, :my_sink]
            perm[b, h, :my_sink] = torch.arange(my_sink, dtype=torch.int32, device=dev)
        dk[b, h, my_sink:my_sink + nr] = x["rows_k"]
        dv[b, h, my_sink:my_sink + nr] = x["rows_v"]
        perm[b, h, my_sink:my_sink + nr] = x["rows_pos"].to(torch.int32)
        if my_window:
            dk[b, h, n_loc - my_window:] = kk[u, nl - my_window:]
            dv[b, h, n_loc - my_window:] = vv[u, nl - my_window:]
            perm[b, h, n_loc - my_window:] = torch.arange(n_tokens - my_window, n_tokens, dtype=torch.int32,
                                                          device=dev)
        nk = c1 - c0
        offs[b, h, 0] = my_sink
        offs[b, h, 1:nk + 1] = my_sink + torch.cumsum(x["counts"], 0).to(torch.int32)
        offs[b, h, nk + 1:] = my_sink + nr
        ncl[b, h] = nk
        cents32[b, h, :nk] = x["cents"][c0:c1].to(torch.float32)
        vbar32[b, h, :nk] = x["vbar"][c0:c1].to(torch.float32)
        gc[b, h, :kc] = x["cents"]
        gv[b, h, :kc] = x["vbar"]
        gs[b, h, :kc] = x["cnt"]
        assignments.append(x["glob_assign"].cpu().numpy())
        objectives.append(x["obj"])
        picks_all.append(x["picks"])
    lay = ClusteredLayer(dk, dv, offs, ncl, cents32, vbar32, perm, n_loc, my_sink, my_window,
                         prefill_tokens=n_loc)
    info = ShardInfo(world=P, rank=r, n_tokens=n_tokens, sink=sink, window=window, k_global=k_glob, c_lo=c_lo,
                     centroids=gc, value_means=gv, sizes=gs, assignment=assignments, objective=objectives,
                     picks=picks_all)
    return lay, info


class SeqShardState:
    """Per-layer step buffers of the sequence-sharded decode (allocated once)."""

    def __init__(self, lay: ClusteredLayer, info: ShardInfo, G: int):
        B, H, cap, d = lay.batch, lay.kv_heads, lay.cluster_cap, lay.head_dim
        dev = lay.device
        Hq = H * G
        self.G = G
        self.rows = B * Hq
        self.ld = int(info.k_global.max())
        self.log_mass = torch.zeros((B, Hq, cap), dtype=torch.float64, device=dev)
        self.state = torch.zeros((B, Hq, cap), dtype=torch.uint8, device=dev)
        self.out = torch.zeros((B, Hq, d), dtype=torch.float32, device=dev)
        self.lse = torch.zeros((B, Hq), dtype=torch.float32, device=dev)
        self.merged = torch.zeros_like(self.out)
        self.merged_lse = torch.zeros_like(self.lse)
        self.g_lm = torch.full((self.rows, self.ld), -math.inf, dtype=torch.float64, device=dev)
        self.g_state = torch.zeros((self.rows, self.ld), dtype=torch.uint8, device=dev)
        self.g_counts = torch.zeros((self.rows, 2), dtype=torch.int32, device=dev)
        kg = np.repeat(info.k_global.reshape(B, H, 1), G, axis=2).reshape(-1).astype(np.int32)
        self.g_k = torch.from_numpy(kg).to(dev)
        self.g_ws = torch.empty((max(N.lib().dp_select_global_workspace_bytes(self.rows, self.ld), 1),),
                                dtype=torch.uint8, device=dev)
        self.ws = torch.zeros((max(N.lib().dp_decode_workspace_bytes(lay.view(), G), 1),), dtype=torch.uint8,
                              device=dev)
        # global cluster id of (rank, local slot) for every row: gather / scatter indices
        P = info.world
        src = np.full((self.rows, self.ld), -1, dtype=np.int64)  # flat index into the all-gathered [P, rows, cap]
        mine_dst = np.full((self.rows, cap), -1, dtype=np.int64)  # global id of my local slot
        for b in range(B):
            for h in range(H):
                for g in range(G):
                    row = (b * H + h) * G + g
                    for rr in range(P):
                        c0, c1 = int(info.c_lo[rr, b, h]), int(info.c_lo[rr + 1, b, h])
                        src[row, c0:c1] = (rr * self.rows + row) * cap + np.arange(c1 - c0)
                    c0, c1 = int(info.c_lo[info.rank, b, h]), int(info.c_lo[info.rank + 1, b, h])
                    mine_dst[row, :c1 - c0] = np.arange(c0, c1)
        valid = src >= 0
        # the same entries in the in-place form's [rows, P * cap] table (slot rr * cap + k)
        self.hole_idx = torch.from_numpy(np.where(valid, (src // cap // self.rows) * cap + src % cap, 0)).to(dev)
        self.src_idx = torch.from_numpy(np.where(valid, src, 0)).to(dev)
        self.src_valid = torch.from_numpy(valid).to(dev)
        mv = mine_dst >= 0
        self.mine_idx = torch.from_numpy(np.where(mv, mine_dst, 0)).to(dev)
        self.mine_valid = torch.from_numpy(mv).to(dev)
        self.cap = cap
        self.use_plan = True  # the fused plan split around the global selection (falls back by shape)
        # in-place form: the selection reads the all-gathered [P, rows, cap] slices directly and the
        # plan reads this rank's states out of the [rows, P * cap] table (no gather / scatter copies)
        self.P = P
        self.in_place = P * cap <= 65536
        self.h_state = torch.zeros((self.rows, P * cap), dtype=torch.uint8, device=dev) if self.in_place else None
        self.h_k = torch.full((self.rows,), P * cap, dtype=torch.int32, device=dev)
        if self.in_place:
            self.h_ws = torch.empty((max(N.lib().dp_select_global_workspace_bytes(self.rows, P * cap), 1),),
                                    dtype=torch.uint8, device=dev)


def seqshard_decode(q, lay: ClusteredLayer, info: ShardInfo, comm: Comm, p1=0.95, p2=0.7, *, state=None,
                    return_plan=False):
    """One decode step of a sequence-sharded layer with global semantics.
    q [B, Hq, d] (identical on every rank).  Returns the merged out [B, Hq, d]
    fp32 on every rank (and the SeqShardState with the global plan)."""
    for name, val in (("p1", p1), ("p2", p2)):
        if not 0.0 < val <= 1.0:
            raise ValueError(f"{name} must be in (0, 1], got {val}")
    B, H = lay.batch, lay.kv_heads
    if q.dim() != 3 or q.shape[0] != B or q.shape[1] % H:
        raise ValueError(f"dimension mismatch: query {tuple(q.shape)}")
    G = q.shape[1] // H
    S = state if state is not None else SeqShardState(lay, info, G)
    q = q.contiguous()
    dev = lay.device
    st = torch.cuda.current_stream(dev).cuda_stream
    lib = N.lib()
    view = lay.view()
    # 1. scores of my cluster slice: the fused plan's scoring phase (dp_plan_score), or
    #    the standalone kernel where the plan does not take the shape
    if S.use_plan:
        rc = lib.dp_plan_score(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass), N.ptr(S.ws),
                               S.ws.numel(), st)
        if rc == N.DP_ERR_UNSUPPORTED:
            S.use_plan = False
        else:
            N.check(rc)
    if not S.use_plan:
        N.check(lib.dp_score(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass), st))
    # 2.-4. in place: the selection reads the all-gathered slices where they landed, the plan reads
    #    my slice's states out of the holey [rows, P * cap] table (dp_plan_score left -inf in the holes)
    if S.use_plan and S.in_place:
        parts = comm.all_gather(S.log_mass.reshape(S.rows, S.cap))  # [P, rows, cap]
        N.check(lib.dp_select_global_parts(N.ptr(parts), S.rows, S.P, S.cap, N.ptr(S.h_k), p1, p2, N.ptr(S.h_state),
                                           N.ptr(S.g_counts), N.ptr(S.h_ws), S.h_ws.numel(), st))
        mine = S.h_state[:, info.rank * S.cap:]
        N.check(lib.dp_plan_given(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass), N.ptr(mine),
                                  S.P * S.cap, None, N.ptr(S.ws), S.ws.numel(), st))
        N.check(lib.dp_attend(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass), N.ptr(S.out),
                              N.ptr(S.lse), N.ptr(S.ws), S.ws.numel(), st))
        if return_plan:  # the global table in global cluster order (as the copying form keeps it)
            S.g_state.copy_(torch.where(S.src_valid, torch.gather(S.h_state, 1, S.hole_idx),
                                        torch.zeros_like(S.g_state)))
        return _merge(S, lay, comm, lib, st, return_plan)
    # 2. the global log-mass table (all-gathered slices, global cluster order)
    parts = comm.all_gather(S.log_mass.reshape(S.rows, S.cap))  # [P, rows, cap]
    flat = parts.reshape(-1)
    S.g_lm.copy_(torch.where(S.src_valid, flat[S.src_idx], torch.full_like(S.g_lm, -math.inf)))
    # 3. global two-stage top-p (identical on every rank)
    N.check(lib.dp_select_global(N.ptr(S.g_lm), S.rows, S.ld, N.ptr(S.g_k), p1, p2, N.ptr(S.g_state),
                                 N.ptr(S.g_counts), N.ptr(S.g_ws), S.g_ws.numel(), st))
    # 4. my slice's states -> local attention over my exact clusters and pseudo-rows
    S.state.reshape(S.rows, S.cap).copy_(torch.where(S.mine_valid, torch.gather(S.g_state, 1, S.mine_idx),
                                                     torch.zeros_like(S.mine_idx, dtype=torch.uint8)))
    if S.use_plan:  # work lists from the given states (cluster-distributed, DSMEM), then the attention grid
        N.check(lib.dp_plan_given(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass), N.ptr(S.state),
                                  0, None, N.ptr(S.ws), S.ws.numel(), st))
        N.check(lib.dp_attend(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass), N.ptr(S.out),
                              N.ptr(S.lse), N.ptr(S.ws), S.ws.numel(), st))
    else:
        N.check(lib.dp_sparse_attention(view, N.ptr(q), dtype_code(q), G, lay.attn_scale, N.ptr(S.log_mass),
                                        N.ptr(S.state), N.ptr(S.out), N.ptr(S.lse), None, N.ptr(S.ws), S.ws.numel(),
                                        st))
    return _merge(S, lay, comm, lib, st, return_plan)


def _merge(S, lay, comm, lib, st, return_plan):
    # 5. the exchange step: all-gather of the partials + the LSE merge kernel
    outs = comm.all_gather(S.out)   # [P, B, Hq, d]
    lses = comm.all_gather(S.lse)   # [P, B, Hq]
    N.check(lib.dp_lse_merge(N.ptr(outs), N.ptr(lses), comm.world, S.rows, lay.head_dim, N.ptr(S.merged),
                             N.ptr(S.merged_lse), st))
    return (S.merged, S) if return_plan else S.merged
