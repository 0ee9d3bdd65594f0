"""Build libdoublep_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2602_05191_b200.build        # or build(force=True)

The library is a plain C-ABI shared object (include/doublep_b200.h) that the
host layer loads with ctypes; no torch headers are involved.
"""

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libdoublep_b200.so")
SOURCES = ["capi.cu", "decode.cu", "cluster.cu", "attn_tc.cu", "plan.cu", "step.cu", "metrics.cu", "shard.cu", "seam.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]
if os.environ.get("DP_PROFILE"):  # %globaltimer phase stamps (tools/plan_timing.py, step_timing.py)
    FLAGS = FLAGS + ["-DDP_PROFILE"]
if os.environ.get("DP_EXTRA_FLAGS"):  # experiment switches, e.g. "-DDP_SEL_REPEAT"
    FLAGS = FLAGS + os.environ["DP_EXTRA_FLAGS"].split()


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _digest():
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)) + ["../../include/doublep_b200.h"]:
        path = os.path.normpath(os.path.join(CSRC, name))
        if os.path.isfile(path):
            h.update(name.encode())
            with open(path, "rb") as f:
                h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(force=False, verbose=False):
    """Compile every .cu for sm_100a and link the shared library (cached by
    source digest).  Returns the library path."""
    os.makedirs(LIBDIR, exist_ok=True)
    stamp = LIB + ".sha256"
    digest = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == digest:
                return LIB
    nvcc = _nvcc()
    objs = []
    logs = []
    procs = []
    for src in SOURCES:  # compiled in parallel
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", path, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src, pr in procs:
        _, err = pr.communicate()
        logs.append(err)
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{err}")
    cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    for o in objs:
        os.remove(o)
    with open(stamp, "w") as f:
        f.write(digest)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
