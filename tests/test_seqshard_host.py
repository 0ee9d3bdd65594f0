"""Host-side pieces of the sequence-sharded path (CPU): the balanced
cluster-range partition and the Comm wrapper over gloo at world size 2
(the collectives seqshard.py issues); the device kernels are covered by
tests/test_gpu_seqshard.py."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_05191_b200 import seqshard as SS


def test_balanced_bounds():
    sizes = np.array([5, 1, 1, 1, 40, 2, 2, 2, 2, 30, 1, 1])
    for world in (1, 2, 3, 4, 12):
        b = SS._balanced_bounds(sizes, world)
        assert b[0] == 0 and b[-1] == sizes.size and np.all(np.diff(b) >= 0) and b.size == world + 1
        cum = np.concatenate([[0], np.cumsum(sizes)])
        for r in range(1, world):  # each boundary is the first cluster reaching r/world of the members
            assert cum[b[r]] >= sizes.sum() * r / world and (b[r] == 0 or cum[b[r] - 1] < sizes.sum() * r / world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = SS.Comm()
        g = c.all_gather(torch.tensor([rank, 10 + rank], dtype=torch.int64))
        s = c.all_reduce(torch.tensor([1.5 * (rank + 1)], dtype=torch.float64))
        m = c.all_reduce(torch.tensor([rank], dtype=torch.int64), op=dist.ReduceOp.MAX)
        q.put((rank, (g.tolist(), float(s.item()), int(m.item()), c.world, c.rank)))
    finally:
        dist.destroy_process_group()


def test_comm_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        g, s, m, w, rk = res[r]
        assert g == [[0, 10], [1, 11]] and s == 4.5 and m == 1 and w == 2 and rk == r
