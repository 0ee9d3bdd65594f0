"""Multi-process (gloo, world size 2) tests of the multi-GPU layout
(SURVEY.md 8e): KV-head shards and the sequence-sharded all-gather LSE merge.
The per-shard attention here is the CPU oracle (tests only); the exchange and
merge are the product code (paper_2602_05191_b200.sharding)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import doublep_oracle as O
from paper_2602_05191_b200 import sharding as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return res


def _case(n=700, d=32, hq=4, seed=3):
    rng = np.random.default_rng(seed)
    keys = rng.normal(size=(n, d)) * 1.5
    values = rng.normal(size=(n, d))
    qs = rng.normal(size=(hq, d)) * 2.0
    return keys, values, qs


def _seq_shard_fn(rank, world):
    keys, values, qs = _case()
    lo, hi = S.seq_shard_bounds(keys.shape[0], world, rank)
    outs, lses = [], []
    for q in qs:
        r = O.full_attention(q, keys[lo:hi], values[lo:hi])
        outs.append(r.output)
        lses.append(r.log_normalizer)
    out = torch.tensor(np.stack(outs), dtype=torch.float32)
    lse = torch.tensor(lses, dtype=torch.float32)
    merged, mlse = S.allgather_lse_merge(out, lse)
    return merged.numpy(), mlse.numpy()


def test_sequence_sharded_merge_equals_full_attention():
    res = _run(_seq_shard_fn)
    keys, values, qs = _case()
    for rank in (0, 1):
        merged, mlse = res[rank]
        for i, q in enumerate(qs):
            ref = O.full_attention(q, keys, values)
            assert O.output_error(merged[i].astype(np.float64), ref.output) <= 1e-5
            assert abs(float(mlse[i]) - ref.log_normalizer) <= 1e-4


def _empty_shard_fn(rank, world):
    keys, values, qs = _case(n=300)
    if rank == 1:  # an empty shard: lse = -inf, out = 0
        out = torch.zeros((qs.shape[0], keys.shape[1]))
        lse = torch.full((qs.shape[0],), -np.inf)
    else:
        out = torch.tensor(np.stack([O.full_attention(q, keys, values).output for q in qs]), dtype=torch.float32)
        lse = torch.tensor([O.full_attention(q, keys, values).log_normalizer for q in qs], dtype=torch.float32)
    merged, _ = S.allgather_lse_merge(out, lse)
    return merged.numpy()


def test_empty_shard_contributes_nothing():
    res = _run(_empty_shard_fn)
    keys, values, qs = _case(n=300)
    for rank in (0, 1):
        for i, q in enumerate(qs):
            assert O.output_error(res[rank][i].astype(np.float64), O.full_attention(q, keys, values).output) <= 1e-5


def _head_shard_fn(rank, world):
    h0, hl = S.kv_head_shard(8, world, rank)
    G, d = 4, 16
    out = torch.arange(hl * G * d, dtype=torch.float32).reshape(1, hl * G, d) + 1000.0 * rank
    full = S.gather_heads(out)
    return (h0, hl, None if full is None else full.numpy())


def test_kv_head_shards_and_gather():
    res = _run(_head_shard_fn)
    assert res[0][:2] == (0, 4) and res[1][:2] == (4, 4)
    full = res[0][2]
    assert full.shape == (1, 32, 16)
    assert full[0, 0, 0] == 0.0 and full[0, 16, 0] == 1000.0
    assert res[1][2] is None


def test_shard_bounds_and_errors():
    n, world = 1_048_576, 8
    bounds = [S.seq_shard_bounds(n, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        S.kv_head_shard(8, 3, 0)


def test_lse_merge_matches_oracle_merge():
    rng = np.random.default_rng(0)
    ms = rng.normal(size=5) * 3
    ls = rng.uniform(0.5, 2.0, size=5)
    os_ = rng.normal(size=(5, 8))
    M, L, o = O.lse_merge(ms, ls, os_)
    # (m, l, o) partials -> (out = o, lse = m + log l)
    out, lse = S.lse_merge(torch.tensor(os_), torch.tensor(ms + np.log(ls)))
    assert np.allclose(out.numpy(), o, atol=1e-12)
    assert abs(float(lse) - (M + np.log(L))) < 1e-5
