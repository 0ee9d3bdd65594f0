"""Golden vectors for the kernel plugin seam, written by the REAL reference's
compiled backend (test infrastructure).

    python oracle/gen_golden_seam.py      # in the build container (baseline/_ref installed)

Calls ``doublep._kernels_cy`` -- the Cython backend of the unmodified
reference installed under baseline/_ref (tools/install_reference.sh;
_kernels_cy.pyx:21-157) -- on seeded inputs shaped like the reference's own
backend-parity tests (tests/test_kernels.py) plus decode-sized ones (d=128,
~1K rows, K=254 centroids), and stores inputs and outputs in
tests/golden/kernels_seam.npz.  tests/test_oracle_golden.py pins the
oracle's Cython-order restatements to it; tests/test_gpu_seam.py checks the
GPU seam (paper_2602_05191_b200.kernels) against it.
"""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

from doublep import _kernels_cy as cy  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "kernels_seam.npz")


def main():
    rng = np.random.default_rng(20260217)
    rec = {}
    # scaled_logits / gather_scaled_logits
    for tag, (n, d, dt) in {"a": (64, 16, np.float32), "b": (64, 16, np.float64), "c": (512, 128, np.float32),
                            "d": (300, 130, np.float64), "e": (1, 5, np.float32)}.items():
        keys = rng.normal(size=(n, d)).astype(dt)
        q = rng.normal(size=d)
        scale = float(1.0 / np.sqrt(d))
        idx = rng.integers(0, n, size=max(1, n // 3)).astype(np.intp)
        rec[f"sl_{tag}_keys"], rec[f"sl_{tag}_q"], rec[f"sl_{tag}_scale"] = keys, q, np.array(scale)
        rec[f"sl_{tag}_idx"] = idx
        rec[f"sl_{tag}_out"] = cy.scaled_logits(keys, q, scale)
        rec[f"sl_{tag}_gout"] = cy.gather_scaled_logits(keys, idx, q, scale)
    # logsumexp / softmax
    for tag, x in {"a": rng.normal(scale=30.0, size=257), "b": np.array([3.25]), "c": rng.normal(size=5000) * 8,
                   "d": np.array([-np.inf, 0.0, -np.inf, 1.0])}.items():
        rec[f"lse_{tag}_x"] = x
        rec[f"lse_{tag}_out"] = np.array(cy.logsumexp(x))
        rec[f"sm_{tag}_out"] = cy.softmax(x)
    # weighted_sum / gather_weighted_sum
    for tag, (n, d, dt) in {"a": (128, 8, np.float32), "b": (1024, 128, np.float32),
                            "c": (513, 64, np.float64)}.items():
        w = rng.random(n)
        mat = rng.normal(size=(n, d)).astype(dt)
        idx = rng.integers(0, n, size=n // 4).astype(np.intp)
        rec[f"ws_{tag}_w"], rec[f"ws_{tag}_mat"], rec[f"ws_{tag}_idx"] = w, mat, idx
        rec[f"ws_{tag}_out"] = cy.weighted_sum(w, mat)
        rec[f"ws_{tag}_gout"] = cy.gather_weighted_sum(w[: idx.shape[0]].copy(), mat, idx)
    # nearest_centroid (random, decode-sized, exact ties)
    cases = {"a": (rng.normal(size=(100, 5)).astype(np.float32), rng.normal(size=(7, 5))),
             "b": (rng.normal(size=(1024, 128)).astype(np.float32), rng.normal(size=(254, 128))),
             "c": (rng.normal(size=(333, 130)), rng.normal(size=(40, 130))),
             "d": (np.zeros((1, 2)), np.array([[1.0, 0.0], [-1.0, 0.0]]))}
    pts = rng.integers(-2, 3, size=(200, 4)).astype(np.float32)  # lattice points: many exact ties
    cents = rng.integers(-2, 3, size=(9, 4)).astype(np.float64)
    cents[5] = cents[2]  # a duplicated centroid: the lower index must win
    cases["e"] = (pts, cents)
    for tag, (p, c) in cases.items():
        a, b = cy.nearest_centroid(p, c)
        rec[f"nc_{tag}_pts"], rec[f"nc_{tag}_cents"] = p, c
        rec[f"nc_{tag}_assign"], rec[f"nc_{tag}_dsq"] = a, b
    # sorted_prefix_count
    vs, ps, counts = [], [], []
    for _ in range(100):
        v = np.sort(rng.random(int(rng.integers(1, 40))))[::-1].copy()
        v /= v.sum()
        p = float(rng.uniform(0.05, 1.0))
        vs.append(v)
        ps.append(p)
        counts.append(cy.sorted_prefix_count(v, p))
    big = np.sort(rng.random(20000) ** 4)[::-1].copy()  # > one 4096-entry GPU chunk
    big /= big.sum()
    rec["spc_big"] = big
    rec["spc_big_p"] = np.array([0.5, 0.9, 0.99, 0.999999, 1.0, 1.5])
    rec["spc_big_count"] = np.array([cy.sorted_prefix_count(big, p) for p in rec["spc_big_p"]])
    rec["spc_lens"] = np.array([len(v) for v in vs])
    rec["spc_vals"] = np.concatenate(vs)
    rec["spc_p"] = np.array(ps)
    rec["spc_count"] = np.array(counts)
    np.savez_compressed(OUT, **rec)
    print("wrote", OUT, len(rec), "arrays")


if __name__ == "__main__":
    main()
