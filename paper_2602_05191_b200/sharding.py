"""Multi-GPU layout of the decode path.

Two ways the path shards across the GPUs of one node, one process per GPU
over ``torch.distributed``:

* **KV-head sharding** (configs 3 and 4).  Rank r owns kv heads
  ``[r*H/P, (r+1)*H/P)`` for every layer and sequence, plus their G q heads.
  Clustering, scoring, selection and attention are all local: there is no
  collective on the decode path; outputs stay head-sharded exactly as in
  tensor-parallel attention (the o-projection all-reduce belongs to the
  model).  ``kv_head_shard`` gives the slice; ``gather_heads`` is the
  validation-only gather of the outputs to one rank.

* **Sequence sharding** (config 5, >= 512K tokens).  Rank r owns the
  contiguous token positions ``seq_shard_bounds(N, P, r)``; each rank runs
  attention over its own tokens and returns a partial (out, lse) per q head;
  ONE exchange step combines them -- an all-gather of (lse, out) followed by
  the log-sum-exp merge (the same math as the split-KV merge inside the
  attention kernel, engine.py:234-246):

      M = max_r lse_r,  w_r = exp(lse_r - M),  out = sum_r w_r out_r / sum_r w_r,
      lse = M + log(sum_r w_r)

  Empty shards contribute lse = -inf.  With dense per-shard attention the
  merged result is exactly full attention over all N tokens.

The exchange works on any backend: NCCL for CUDA tensors (NVLink), gloo for
the CPU tests (tests/test_sharding.py, world size 2).
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist


def kv_head_shard(kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(first kv head, kv heads) owned by `rank` under KV-head sharding."""
    if kv_heads % world:
        raise ValueError(f"kv heads {kv_heads} not divisible by {world} ranks")
    per = kv_heads // world
    return rank * per, per


def seq_shard_bounds(n_tokens: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous token positions [lo, hi) owned by `rank` (balanced to +-1)."""
    return n_tokens * rank // world, n_tokens * (rank + 1) // world


def lse_merge(out: torch.Tensor, lse: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Merge P partials: out [P, ..., d], lse [P, ...] -> (out [..., d], lse [...]).

    Partials with lse = -inf (empty shards) get weight 0; if every partial is
    empty the result is out = 0, lse = -inf."""
    lse = lse.to(torch.float64)
    m = lse.max(dim=0).values
    finite = torch.isfinite(m)
    m_safe = torch.where(finite, m, torch.zeros_like(m))
    w = torch.exp(lse - m_safe.unsqueeze(0))
    w = torch.where(torch.isfinite(lse), w, torch.zeros_like(w))
    tot = w.sum(dim=0)
    merged = (w.unsqueeze(-1) * out.to(torch.float64)).sum(dim=0) / torch.where(
        tot > 0, tot, torch.ones_like(tot)).unsqueeze(-1)
    merged_lse = torch.where(tot > 0, m_safe + torch.log(torch.where(tot > 0, tot, torch.ones_like(tot))),
                             torch.full_like(tot, -math.inf))
    return merged.to(out.dtype), merged_lse.to(torch.float32)


def allgather_lse_merge(out: torch.Tensor, lse: torch.Tensor, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Sequence-sharded exchange step: every rank contributes its partial
    (out [..., d], lse [...]) and receives the merged (out, lse).  One
    all-gather of lse and of out (NCCL over NVLink for CUDA tensors)."""
    world = dist.get_world_size(group)
    if world == 1:
        return out, lse
    lse = lse.contiguous().to(torch.float32)
    out = out.contiguous()
    lses = [torch.empty_like(lse) for _ in range(world)]
    outs = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(lses, lse, group=group)
    dist.all_gather(outs, out, group=group)
    return lse_merge(torch.stack(outs), torch.stack(lses))


def gather_heads(out: torch.Tensor, group=None, dst: int = 0):
    """Validation only (outside any timed region): collect head-sharded
    outputs [B, Hq/P, d] from all ranks into [B, Hq, d] on `dst`."""
    world = dist.get_world_size(group)
    if world == 1:
        return out
    parts = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(parts, out.contiguous(), group=group)
    return torch.cat(parts, dim=1) if dist.get_rank(group) == dst else None


def sequence_sharded_attention(q: torch.Tensor, layer_shard, group=None, *, sparse: bool = True, p1: float = 0.95,
                               p2: float = 0.7, workspace=None):
    """Decode step over a sequence-sharded layer: local attention over this
    rank's tokens (the rank's own ClusteredLayer -- sparse Double-P or the
    dense kernel), then the all-gather LSE merge.  Returns the merged
    out [B, Hq, d] fp32 on every rank."""
    from .engine import dense_attention, sparse_attention

    if sparse:
        out, ws = sparse_attention(q, layer_shard, p1, p2, workspace=workspace, return_plan=True)
        lse = ws.lse
    else:
        out, lse = dense_attention(q, layer_shard, workspace=workspace, return_lse=True)
    merged, _ = allgather_lse_merge(out, lse, group)
    return merged
