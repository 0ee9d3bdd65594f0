"""Golden DPKV file written by the REAL reference (test infrastructure).

    python oracle/gen_golden_dpkv.py      # in the build container (/root/reference present)

Uses doublep.workload.generate + doublep.kvcache.write_dump (kvcache.py:156-192)
and stores, next to the file, the arrays read_dump returns, so
tests/test_dpkv.py can check paper_2602_05191_b200.dpkv against the
reference's own writer and reader without /root/reference at run time.
"""
import os
import sys

import numpy as np

os.environ["DOUBLEP_KERNELS"] = "python"
sys.path.insert(0, "/root/reference/pkg/src")

from doublep import kvcache, workload  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main():
    spec = workload.WorkloadSpec(context_len=96, head_dim=16, num_layers=2, num_kv_heads=2, gqa_group=2,
                                 num_steps=2, tail_profile="mixed", seed=7)
    cache, trace = workload.generate(spec)
    path = os.path.join(OUT, "ref_small.dpkv")
    kvcache.write_dump(cache, trace, path)
    c2, t2 = kvcache.read_dump(path)
    np.savez(os.path.join(OUT, "ref_small_dpkv.npz"), keys=c2.keys, values=c2.values, queries=t2.queries,
             gqa_group=t2.gqa_group)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
