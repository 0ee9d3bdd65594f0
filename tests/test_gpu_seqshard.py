"""Sequence-sharded Double-P with global semantics (config 5):
two ranks (gloo, both on cuda:0) each hold half of the token positions; the
sharded prefill clustering, the global two-stage top-p and the LSE-merged
output must equal the UNSHARDED oracle (oracle/doublep_oracle.py, the
reference's algorithm) -- k-means++ picks and Lloyd assignments of the whole
sequence, the selection sets of the global cluster table (ties classified,
tests/parity.py) and the outputs within the fp32 tolerance."""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import doublep_oracle as O
import parity as PT

pytestmark = pytest.mark.gpu

N_TOK, D, H, G, SINK, WIN = 3000, 64, 2, 4, 4, 64


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spec(profile):
    return O.WorkloadSpec(context_len=N_TOK, head_dim=D, num_kv_heads=H, gqa_group=G, num_steps=3,
                          tail_profile=profile, seed=0)


def _worker(rank, world, port, profile, p1, p2, q_out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_05191_b200 import seqshard as SS
        from paper_2602_05191_b200.sharding import seq_shard_bounds

        torch.cuda.set_device(0)
        keys, values, queries = O.generate(_spec(profile))
        lo, hi = seq_shard_bounds(N_TOK, world, rank)
        k = torch.from_numpy(keys[0][None, :, lo:hi]).cuda()
        v = torch.from_numpy(values[0][None, :, lo:hi]).cuda()
        comm = SS.Comm()
        lay, info = SS.shard_cluster_layer(k, v, N_TOK, comm, sink=SINK, window=WIN, seed=0)
        outs, states, counts = [], [], []
        st = None
        for s in range(queries.shape[0]):
            q = torch.from_numpy(queries[s, 0][None]).cuda()
            out, st = SS.seqshard_decode(q, lay, info, comm, p1, p2, state=st, return_plan=True)
            torch.cuda.synchronize()
            outs.append(out[0].double().cpu().numpy())
            states.append(st.g_state.cpu().numpy().copy())
            counts.append(st.g_counts.cpu().numpy().copy())
        res = dict(picks=info.picks, assign=info.assignment, objective=info.objective,
                   cents=info.centroids.cpu().numpy(), vbar=info.value_means.cpu().numpy(),
                   sizes=info.sizes.cpu().numpy(), kglob=info.k_global, outs=outs, states=states, counts=counts)
        q_out.put((rank, res))
    except Exception as e:  # surfaced by the parent
        import traceback

        q_out.put((rank, traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, profile, p1, p2):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, profile, p1, p2, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r, x in res.items():
        assert isinstance(x, dict), f"rank {r} failed:\n{x}"
    return res


@pytest.mark.parametrize("profile,p1,p2", [("peaked", 0.95, 0.7), ("mixed", 0.9, 0.8)])
def test_sequence_sharded_global_semantics(profile, p1, p2):
    world = 2
    res = _run(world, profile, p1, p2)
    r0 = res[0]
    for r in range(1, world):  # every rank derived the same global tables and plan
        np.testing.assert_array_equal(res[r]["kglob"], r0["kglob"])
        for a, b in zip(res[r]["states"], r0["states"]):
            np.testing.assert_array_equal(a, b)
        for a, b in zip(res[r]["outs"], r0["outs"]):
            np.testing.assert_array_equal(a, b)
    keys, values, queries = O.generate(_spec(profile))
    k = O.default_cluster_count(N_TOK - SINK - WIN)
    agree_min, classes = 1.0, {"exact": 0, "order_tie": 0, "threshold_tie": 0, "real": 0}
    worst = 0.0
    for h in range(H):
        mid = keys[0, h, SINK:N_TOK - WIN]
        # --- clustering vs the unsharded reference algorithm
        x64 = mid.astype(np.float64)
        cent0, picks0 = O.plusplus_init(x64, k, np.random.default_rng(O.head_seed(0, 0, h)))
        np.testing.assert_array_equal(r0["picks"][h], picks0)  # k-means++ picks: bit-exact
        fit = O.lloyd(mid, cent0, 25)
        kg = int(r0["kglob"][0, h])
        assert kg == fit.centroids.shape[0]
        agree = float(np.mean(r0["assign"][h] == fit.assignments))
        agree_min = min(agree_min, agree)
        assert agree >= 1 - 1e-3, agree
        assert abs(r0["objective"][h][-1] - fit.objective[-1]) <= 1e-5 * fit.objective[-1]
        # --- decode: the oracle fed the sharded build's GLOBAL tables
        members = [np.flatnonzero(r0["assign"][h] == c).astype(np.int64) + SINK for c in range(kg)]
        tables = O.HeadTables(members=members, centroids=r0["cents"][0, h, :kg].astype(np.float32).astype(np.float64),
                              value_means=r0["vbar"][0, h, :kg].astype(np.float32).astype(np.float64))
        for s in range(queries.shape[0]):
            for g in range(G):
                hq = h * G + g
                qv = queries[s, 0, hq].astype(np.float64)
                ref, pl, est = O.decode_step(qv, keys[0, h].astype(np.float64), values[0, h].astype(np.float64),
                                             tables, p1, p2, SINK, WIN)
                st_row = r0["states"][s][hq][:kg]
                c1, c2 = PT.classify_sets(est, pl, st_row, p1, p2)
                classes[c1] += 1
                classes[c2] += 1
                assert "real" not in (c1, c2), (h, s, g, c1, c2)
                if (c1, c2) == ("exact", "exact"):
                    err = O.output_error(r0["outs"][s][hq], ref.output)
                    worst = max(worst, err)
                    assert err <= 1e-5, err
    print(f"[SEQSHARD] {profile} p=({p1},{p2}) world {world}: k-means assignment agreement >= {agree_min:.6f}, "
          f"stage classes {classes}, worst rel err {worst:.2e}")


def test_lse_merge_kernel():
    """dp_lse_merge against the fp64 host merge (empty partials included)."""
    from paper_2602_05191_b200 import _native as N

    g = torch.Generator().manual_seed(0)
    P, rows, d = 3, 5, 64
    outs = torch.randn((P, rows, d), generator=g)
    lses = torch.randn((P, rows), generator=g) * 5
    lses[1, 2] = -float("inf")
    lses[:, 4] = -float("inf")  # a row with no mass anywhere
    o_d, l_d = outs.cuda(), lses.cuda()
    out = torch.zeros((rows, d), device="cuda")
    lse = torch.zeros((rows,), device="cuda")
    N.check(N.lib().dp_lse_merge(N.ptr(o_d), N.ptr(l_d), P, rows, d, N.ptr(out), N.ptr(lse),
                                 torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    L = lses.double()
    M = L.max(dim=0).values
    Ms = torch.where(torch.isfinite(M), M, torch.zeros_like(M))
    w = torch.where(torch.isfinite(L), torch.exp(L - Ms), torch.zeros_like(L))
    tot = w.sum(0)
    ref = (w.unsqueeze(-1) * outs.double()).sum(0) / torch.where(tot > 0, tot, torch.ones_like(tot)).unsqueeze(-1)
    assert torch.allclose(out.cpu().double()[:4], ref[:4], rtol=1e-6, atol=1e-6)
    assert torch.all(out.cpu()[4] == 0) and lse.cpu()[4].item() == -float("inf")
    assert torch.allclose(lse.cpu().double()[:4], (Ms + torch.log(tot))[:4], rtol=1e-6, atol=1e-6)


def test_select_global_matches_fused_plan():
    """dp_select_global (any K) reproduces the per-head states of dp_select on
    the same log-masses."""
    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200 import cluster_layer
    from paper_2602_05191_b200.workload import generate_layer, generate_queries

    k, v, c = generate_layer(1, 2, 8192, 128)
    lay = cluster_layer(k, v, fp64_assign=False)
    q = torch.from_numpy(generate_queries(c, 4, 1)[0]).cuda().to(torch.bfloat16)
    cap = lay.cluster_cap
    lm = torch.zeros((1, 8, cap), dtype=torch.float64, device="cuda")
    st_ref = torch.zeros((1, 8, cap), dtype=torch.uint8, device="cuda")
    cnt_ref = torch.zeros((1, 8, 2), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    lib = N.lib()
    N.check(lib.dp_score(lay.view(), N.ptr(q), 1, 4, lay.attn_scale, N.ptr(lm), s))
    ws = torch.zeros((lib.dp_decode_workspace_bytes(lay.view(), 4),), dtype=torch.uint8, device="cuda")
    N.check(lib.dp_select(lay.view(), 4, 0.95, 0.7, N.ptr(lm), N.ptr(st_ref), N.ptr(cnt_ref), None, None, None,
                          N.ptr(ws), ws.numel(), s))
    ks = lay.nclusters.repeat_interleave(4, dim=1).reshape(-1).to(torch.int32)
    st = torch.zeros((8, cap), dtype=torch.uint8, device="cuda")
    cnt = torch.zeros((8, 2), dtype=torch.int32, device="cuda")
    gws = torch.empty((lib.dp_select_global_workspace_bytes(8, cap),), dtype=torch.uint8, device="cuda")
    N.check(lib.dp_select_global(N.ptr(lm), 8, cap, N.ptr(ks), 0.95, 0.7, N.ptr(st), N.ptr(cnt), N.ptr(gws),
                                 gws.numel(), s))
    torch.cuda.synchronize()
    for r in range(8):
        kk = int(ks[r])
        assert torch.equal(st[r, :kk], st_ref[0, r, :kk]), r
        assert torch.equal(cnt[r], cnt_ref[0, r]), r


@pytest.mark.parametrize("K", [32766, 50000])
def test_select_global_large_k_vs_oracle(K):
    """The global table of the 1M-token config (K = 32,766; beyond the fused
    plan's and dp_select's per-launch caps): dp_select_global against the
    oracle's two-stage top-p (selection.py:36-65) on peaked and flat rows,
    ties classified as in tests/parity.py."""
    from types import SimpleNamespace

    from paper_2602_05191_b200 import _native as N

    rng = np.random.default_rng(7)
    rows = []
    for kind in ("peaked", "flat", "two-peak"):
        base = rng.normal(0.0, 1.0, K) + np.log(rng.integers(1, 80, K))
        if kind == "peaked":
            base[rng.integers(0, K, 300)] += rng.uniform(4, 14, 300)
        elif kind == "two-peak":
            base[:50] += 20.0
            base[-50:] += 19.5
        rows.append(base * (0.3 if kind == "flat" else 1.0))
    lm = torch.from_numpy(np.stack(rows)).cuda()
    R = lm.shape[0]
    ks = torch.full((R,), K, dtype=torch.int32, device="cuda")
    st = torch.zeros((R, K), dtype=torch.uint8, device="cuda")
    cnt = torch.zeros((R, 2), dtype=torch.int32, device="cuda")
    lib = N.lib()
    for p1, p2 in ((0.95, 0.7), (0.9, 0.8), (0.99, 0.5)):
        ws = torch.empty((lib.dp_select_global_workspace_bytes(R, K),), dtype=torch.uint8, device="cuda")
        N.check(lib.dp_select_global(N.ptr(lm), R, K, N.ptr(ks), p1, p2, N.ptr(st), N.ptr(cnt), N.ptr(ws),
                                     ws.numel(), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        for r in range(R):
            x = rows[r]
            probs = O.softmax(x)
            est = SimpleNamespace(probs=probs)
            s1 = O.top_p_select(probs, p1)
            pl = SimpleNamespace(stage1=s1)
            c1, c2 = PT.classify_sets(est, pl, st[r].cpu().numpy(), p1, p2)
            assert "real" not in (c1, c2), (r, p1, p2, c1, c2)
            n1 = int((st[r] >= 1).sum())
            assert int(cnt[r, 0]) == n1 and int(cnt[r, 1]) == int((st[r] == 2).sum())


@pytest.mark.parametrize("K", [700, 8192, 20000, 32766, 50000])
def test_select_global_paths_identical(K):
    """The one-launch clustered selection (DSMEM exchanges, the default up to
    K = 65,536), the five-launch split form and the one-CTA-per-row kernel
    give bit-identical states and counts -- including rows so flat that the
    candidates overflow shared memory into global scratch, rows with -inf /
    NaN entries, exact ties and ragged per-row K."""
    from paper_2602_05191_b200 import _native as N

    rng = np.random.default_rng(K)
    rows = []
    for kind in ("peaked", "flat", "ties", "nonfinite", "tiny"):
        base = rng.normal(0.0, 1.0, K) + np.log(rng.integers(1, 80, K))
        if kind == "peaked":
            base[rng.integers(0, K, max(1, K // 100))] += rng.uniform(4, 14, max(1, K // 100))
        elif kind == "flat":
            base = base * 0.01
        elif kind == "ties":
            base = np.round(base * 4) / 4
        elif kind == "nonfinite":
            base[rng.integers(0, K, 50)] = -np.inf
            base[rng.integers(0, K, 5)] = np.nan
        else:
            base = np.full(K, -np.inf)
        rows.append(base)
    lm = torch.from_numpy(np.stack(rows)).cuda()
    R = lm.shape[0]
    ks = torch.tensor([K, K, max(1, K - 3), K, K], dtype=torch.int32, device="cuda")
    lib = N.lib()
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.empty((lib.dp_select_global_workspace_bytes(R, K),), dtype=torch.uint8, device="cuda")
    res = {}
    try:
        for path in (3, 1, 2):
            if path == 3 and K > 65536:
                continue
            lib.dp_debug_set(11, path)
            for p1, p2 in ((0.95, 0.7), (0.5, 0.9), (1.0, 0.7), (1.0, 1.0)):
                st = torch.full((R, K), 9, dtype=torch.uint8, device="cuda")
                cnt = torch.zeros((R, 2), dtype=torch.int32, device="cuda")
                N.check(lib.dp_select_global(N.ptr(lm), R, K, N.ptr(ks), p1, p2, N.ptr(st), N.ptr(cnt), N.ptr(ws),
                                             ws.numel(), s))
                torch.cuda.synchronize()
                res[(path, p1, p2)] = (st.cpu(), cnt.cpu())
    finally:
        lib.dp_debug_set(11, 0)
    for (path, p1, p2), (st, cnt) in res.items():
        ref_st, ref_cnt = res[(2, p1, p2)]
        for r in range(R):
            kk = int(ks[r])
            assert torch.equal(st[r, :kk], ref_st[r, :kk]), (path, p1, p2, r)
            assert int(cnt[r, 0]) == int((st[r, :kk] >= 1).sum()) and int(cnt[r, 1]) == int((st[r, :kk] == 2).sum())
        assert torch.equal(cnt, ref_cnt), (path, p1, p2)


@pytest.mark.parametrize("P,part_len", [(2, 700), (8, 4096), (5, 3000)])
def test_select_global_parts_in_place(P, part_len):
    """dp_select_global_parts reads the all-gathered [P, rows, part_len]
    slices in place (holes at -inf, as dp_plan_score leaves them): the same
    states and counts as dp_select_global on the flattened global table."""
    from paper_2602_05191_b200 import _native as N

    rng = np.random.default_rng(P * 1000 + part_len)
    R = 6
    parts = rng.normal(0.0, 1.0, (P, R, part_len)) + np.log(rng.integers(1, 80, (P, R, part_len)))
    parts[:, :, rng.integers(0, part_len, 40)] += 9.0
    for p in range(P):  # ragged slices: each rank holds fewer clusters than the slot count
        n_p = int(rng.integers(part_len // 2, part_len + 1))
        parts[p, :, n_p:] = -np.inf
    parts[:, 3] = np.round(parts[:, 3] * 2) / 2  # exact ties across slices
    flat = np.ascontiguousarray(parts.transpose(1, 0, 2).reshape(R, P * part_len))
    lib = N.lib()
    s = torch.cuda.current_stream().cuda_stream
    K = P * part_len
    t_parts = torch.from_numpy(np.ascontiguousarray(parts)).cuda()
    t_flat = torch.from_numpy(flat).cuda()
    ks = torch.full((R,), K, dtype=torch.int32, device="cuda")
    ws = torch.empty((lib.dp_select_global_workspace_bytes(R, K),), dtype=torch.uint8, device="cuda")
    for p1, p2 in ((0.95, 0.7), (0.6, 0.9), (1.0, 0.5)):
        st_a = torch.zeros((R, K), dtype=torch.uint8, device="cuda")
        st_b = torch.zeros((R, K), dtype=torch.uint8, device="cuda")
        c_a = torch.zeros((R, 2), dtype=torch.int32, device="cuda")
        c_b = torch.zeros((R, 2), dtype=torch.int32, device="cuda")
        N.check(lib.dp_select_global(N.ptr(t_flat), R, K, N.ptr(ks), p1, p2, N.ptr(st_a), N.ptr(c_a), N.ptr(ws),
                                     ws.numel(), s))
        N.check(lib.dp_select_global_parts(N.ptr(t_parts), R, P, part_len, N.ptr(ks), p1, p2, N.ptr(st_b),
                                           N.ptr(c_b), N.ptr(ws), ws.numel(), s))
        torch.cuda.synchronize()
        assert torch.equal(st_a, st_b), (p1, p2)
        assert torch.equal(c_a, c_b), (p1, p2)
