"""Parity helpers shared by the GPU tests: feed the oracle the GPU's own
tables (SURVEY.md §8c protocol step 1) and classify selection mismatches
(order tie / threshold tie / real, step 2)."""

import numpy as np

from oracle import doublep_oracle as O

TIE = 1e-6


def oracle_tables(layer, b, h):
    """The GPU's clustered tables of one head as an oracle HeadTables."""
    t = layer.head_tables(b, h)
    return O.HeadTables(members=t["members"], centroids=t["centroids"], value_means=t["value_means"])


def classify_stage(probs_o, order_o, n_o, order_g, n_g, cum_o, p):
    """Compare one top-p stage of the oracle (order_o, n_o, normalised
    cumulative mass cum_o) with the GPU's (order_g, n_g).  Returns 'exact',
    'order_tie', 'threshold_tie' or 'real'."""
    a = np.asarray(order_o[:n_o])
    g = np.asarray(order_g[:n_g])
    if n_o == n_g and np.array_equal(a, g):
        return "exact"
    scale = max(float(np.max(probs_o)), 1e-300)
    for i in range(min(n_o, n_g)):
        if a[i] != g[i] and abs(probs_o[a[i]] - probs_o[g[i]]) > TIE * scale:
            return "real"
    if n_o == n_g:
        return "order_tie"
    lo, hi = sorted((n_o, n_g))
    for j in range(lo - 1, hi - 1):
        if abs(cum_o[j] - p) > TIE:
            return "real"
    return "threshold_tie"


def compare_plan(est_o, plan_o, order_g, n1_g, n2_g, p1, p2):
    """Classify stage 1 and stage 2 of one (q head) plan."""
    probs = est_o.probs
    order_o = np.argsort(-probs, kind="stable")
    cum1 = np.cumsum(probs[order_o]) / probs.sum()
    n1_o = plan_o.stage1.selected.size
    n2_o = plan_o.exact_clusters.size
    c1 = classify_stage(probs, order_o, n1_o, order_g, n1_g, cum1, p1)
    sub = probs[order_o[:n1_o]]
    cum2 = np.cumsum(sub) / sub.sum()
    c2 = classify_stage(probs, order_o, n2_o, order_g, n2_g, cum2, p2) if c1 == "exact" else c1
    return c1, c2


def _same_modulo_ties(probs, got, want, scale):
    """Sets `got` and `want` (equal size) hold the same probabilities up to
    swaps of entries within TIE*scale of each other."""
    a = np.sort(probs[np.asarray(sorted(got - want), dtype=np.int64)]) if got - want else np.empty(0)
    b = np.sort(probs[np.asarray(sorted(want - got), dtype=np.int64)]) if want - got else np.empty(0)
    return a.size == b.size and np.all(np.abs(a - b) <= TIE * scale)


def classify_sets(est_o, plan_o, state_row, p1, p2):
    """Classify the GPU plan given as per-cluster states (2 exact, 1 approx,
    0 dropped) against the oracle plan: 'exact', 'order_tie',
    'threshold_tie' or 'real' for each stage."""
    probs = est_o.probs
    K = probs.size
    st = np.asarray(state_row[:K])
    order = np.argsort(-probs, kind="stable")
    scale = max(float(probs.max()), 1e-300)
    res = []
    for stage in (1, 2):
        if stage == 1:
            g = set(np.flatnonzero(st >= 1).tolist())
            o_set = set(plan_o.stage1.selected.tolist())
            cum = np.cumsum(probs[order]) / probs.sum()
            p = p1
            base = order
        else:
            g = set(np.flatnonzero(st == 2).tolist())
            # stage 2 runs on the stage-1 set actually selected; after a
            # stage-1 tie that is the GPU's set, so re-derive the oracle cut
            n1 = plan_o.stage1.selected.size if res[0] == "exact" else int((st >= 1).sum())
            sub = probs[order[:n1]]
            cum = np.cumsum(sub) / sub.sum()
            n2 = min(int(np.searchsorted(cum, p2, side="left")) + 1, n1)
            o_set = set(order[:n2].tolist())
            p = p2
            base = order[:n1]
        if g == o_set:
            res.append("exact")
            continue
        ng, no = len(g), len(o_set)
        if not _same_modulo_ties(probs, g, set(base[:ng].tolist()), scale):
            res.append("real")
            continue
        if ng == no:
            res.append("order_tie")
            continue
        lo, hi = sorted((ng, no))
        res.append("threshold_tie" if all(abs(cum[j] - p) <= TIE for j in range(lo - 1, hi - 1)) else "real")
    return tuple(res)
