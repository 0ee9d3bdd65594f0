"""Device-side synthetic KV caches with the reference's generator law.

Reference law: /root/reference/pkg/src/doublep/workload.py:130-194 -- keys
are Gaussian blobs (centres ~ N(0, separation), per-token blob uniform,
spread N(0, 0.3)), values share the blob structure (vcentres ~ N(0, 1) +
N(0, 0.5)), queries aim at the blobs by tail profile ("peaked": one blob at
gain 3*U(1,1.3)*sqrt(d) 75% of the time, a multi-blob minimum-norm direction
otherwise; "heavy": several blobs at gain 3.7*U(0.75,1.25)*sqrt(d);
"uniform": zero query; "mixed": round-robin per head).

Host generation of 32 layers x 8 heads x 32K-128K rows takes minutes, so the
K/V draws use torch's device RNG (Philox) with the same distributions; the
small query directions are computed on the host with NumPy.  The exact
reference streams are reproduced only by the CPU oracle (tests use that).
"""

from __future__ import annotations

import numpy as np
import torch

PROFILES = ("peaked", "heavy", "uniform", "mixed")


def _unit(v):
    n = np.linalg.norm(v)
    return v if n == 0.0 else v / n


def _multi_blob_direction(centers, chosen):
    """Minimum-norm direction with equal projection on the chosen centres
    and leak suppression (`workload.py:104-127`)."""
    dim = centers.shape[1]
    chosen = list(chosen)
    suppressed = []
    while True:
        rows = centers[chosen + suppressed]
        targets = np.concatenate([np.ones(len(chosen)), np.zeros(len(suppressed))])
        u, *_ = np.linalg.lstsq(rows, targets, rcond=None)
        u = _unit(u)
        level = float(np.mean(centers[chosen] @ u))
        taken = set(chosen) | set(suppressed)
        others = [b for b in range(len(centers)) if b not in taken]
        if not others or len(taken) >= dim - 2:
            return u
        leaks = centers[others] @ u
        worst = int(np.argmax(leaks))
        if leaks[worst] <= 0.55 * level:
            return u
        suppressed.append(others[worst])


def _query(rng, centers, profile, d, num_blobs):
    if profile == "peaked":
        if rng.random() < 0.25:
            count = min(max(2, num_blobs // 3), len(centers))
            direction = _multi_blob_direction(centers, rng.choice(len(centers), size=count, replace=False))
        else:
            direction = _unit(centers[int(rng.integers(len(centers)))])
        return 3.0 * rng.uniform(1.0, 1.3) * np.sqrt(d) * direction
    if profile == "heavy":
        count = min(max(2, num_blobs // 4), len(centers))
        chosen = rng.choice(len(centers), size=count, replace=False)
        direction = _unit(np.sum([_unit(centers[b]) for b in chosen], axis=0))
        return 3.7 * rng.uniform(0.75, 1.25) * np.sqrt(d) * direction
    return np.zeros(d)


def generate_layer(batch, kv_heads, context, head_dim, *, layer=0, seed=0, num_blobs=8, blob_spread=0.3,
                   blob_separation=1.0, dtype=torch.bfloat16, device="cuda"):
    """Keys/values [B,H,N,d] (dtype) and blob centres [B,H,blobs,d] (fp64 host)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence([seed, 0xD0B1E, layer]).generate_state(1)[0]))
    B, H, N, d = batch, kv_heads, context, head_dim
    centers = torch.randn((B, H, num_blobs, d), generator=g, device=device, dtype=torch.float32) * blob_separation
    vcenters = torch.randn((B, H, num_blobs, d), generator=g, device=device, dtype=torch.float32)
    assign = torch.randint(0, num_blobs, (B, H, N), generator=g, device=device)
    idx = assign.unsqueeze(-1).expand(B, H, N, d)
    keys = torch.randn((B, H, N, d), generator=g, device=device, dtype=torch.float32).mul_(blob_spread)
    keys.add_(torch.gather(centers, 2, idx))
    values = torch.randn((B, H, N, d), generator=g, device=device, dtype=torch.float32).mul_(0.5)
    values.add_(torch.gather(vcenters, 2, idx))
    del idx, assign
    return keys.to(dtype), values.to(dtype), centers.double().cpu().numpy()


def generate_queries(centers, gqa_group, steps, *, profile="peaked", layer=0, seed=0, num_blobs=8):
    """Queries [steps, B, H*G, d] fp32 (host numpy) aimed at the blob centres."""
    B, H, _, d = centers.shape
    Hq = H * gqa_group
    out = np.zeros((steps, B, Hq, d), dtype=np.float32)
    cycle = ("peaked", "heavy", "uniform")
    for b in range(B):
        for hq in range(Hq):
            rng = np.random.default_rng(np.random.SeedSequence([seed, 2, layer, hq, b]))
            prof = profile if profile != "mixed" else cycle[(layer * Hq + hq) % 3]
            for s in range(steps):
                out[s, b, hq] = _query(rng, centers[b, hq // gqa_group], prof, d, num_blobs)
    return out
