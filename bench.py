#!/usr/bin/env python
"""Double-P decode-step benchmark (driver contract).

Workload (BASELINE.json configs[1]): Llama-3.1-8B-shaped decode, 32 layers,
batch 1, 32K context, 8 KV heads x 4 q heads (GQA 4), head_dim 128, bf16
cache, (p1, p2) = (0.95, 0.7), synthetic blob KV caches with the reference's
generator law ("peaked" queries).  One step = one decode step of every layer
(score -> select -> worklist -> gathered split-KV attention + LSE merge),
layers run back to back from HBM (each layer's cache is 134 MB > L2, so no
flush is needed between steps).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): KV heads are sharded across ranks (strong scaling),
no collective on the data path; time = max over ranks.
"""

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--context", type=int, default=32768)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--gqa", type=int, default=4)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--p1", type=float, default=0.95)
    ap.add_argument("--p2", type=float, default=0.7)
    ap.add_argument("--profile", default="peaked")
    ap.add_argument("--qsteps", type=int, default=8, help="distinct query steps cycled through")
    ap.add_argument("--fp64-assign", type=int, default=0, help="prefill k-means distances in fp64")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-fi-dense", action="store_true", help="skip the flashinfer trtllm-gen dense comparator")
    ap.add_argument("--mixed-layers", type=int, default=8,
                    help="layers of the 'mixed' stress-profile line at the headline context (0: off)")
    ap.add_argument("--cpu-sample-heads", type=int, default=2)
    ap.add_argument("--long-context", type=int, default=131072,
                    help="secondary workload context (0: off); reported under long_context")
    ap.add_argument("--long-layers", type=int, default=4)
    ap.add_argument("--prefill-group-gib", type=float, default=16.0,
                    help="position-ordered KV clustered per launch (bounds the prefill's transient memory)")
    ap.add_argument("--sim-world", type=int, default=1,
                    help="measure ONE rank's KV-head shard of a P-GPU run on this GPU (no collectives)")
    ap.add_argument("--sim-rank", type=int, default=0)
    ap.add_argument("--seq-shards", type=int, default=1,
                    help="config 5: shard the sequence over P ranks (global two-stage top-p over the "
                         "all-gathered log-mass slices + LSE merge); under torchrun P = world, else one "
                         "rank's share (--sim-rank) is measured alone on one GPU")
    return ap.parse_args()


def model_name(a):
    return "llama-3.1-8b-shape" if a.kv_heads * a.gqa == 32 else ("llama-3.1-70b-shape" if a.gqa == 8 else "custom")


def workload_config(a, world):
    return {
        "workload": f"doublep-decode {model_name(a)} L{a.layers} B{a.batch} N{a.context} "
                    f"Hq{a.kv_heads * a.gqa}/Hkv{a.kv_heads} d{a.head_dim} bf16 p=({a.p1},{a.p2}) {a.profile}",
        "layers": a.layers, "batch": a.batch, "context": a.context, "kv_heads": a.kv_heads,
        "q_heads": a.kv_heads * a.gqa, "head_dim": a.head_dim, "p1": a.p1, "p2": a.p2,
        "tail_profile": a.profile, "sink": 4, "window": 64, "tokens_per_cluster": 32,
        "parallelism": (f"kv-head shard x{world}" if world > 1 else
                        (f"kv-head shard {a.sim_rank}/{a.sim_world} measured alone on one GPU (per-GPU share of a "
                         f"{a.sim_world}-GPU run)" if a.sim_world > 1 else "single GPU")),
        "l2": "inputs larger than L2 (each layer's KV > 126 MB; layers cycled)",
    }


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_setup():
    """(world, rank, local device).  DP_SAME_DEVICE=1 runs every rank on
    cuda:0 over gloo -- a plumbing dry run of an N-GPU launch on one GPU."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    same = os.environ.get("DP_SAME_DEVICE") == "1"
    if same:
        local = 0
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if _cuda() and not same else "gloo")
    return world, rank, local


def _cuda():
    import torch

    return torch.cuda.is_available()


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=device if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------------------
# CPU reference: the UNMODIFIED reference package (doublep 0.1.0, installed at
# baseline/_ref by tools/install_reference.sh) timed on the host cores -- a
# reported baseline only.  Each backend configuration runs in its own process
# (the backend is chosen at import, kernels.py:17-29; BLAS threads at load).
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

_REF_WORKER = r"""
import json, pickle, sys, time
sys.path.insert(0, sys.argv[1])
import doublep
from doublep import engine
with open(sys.argv[2], "rb") as f:
    job = pickle.load(f)
cache, cc, calls = job["cache"], job["cc"], job["calls"]
cfg = engine.DoublePConfig(job["p1"], job["p2"], sink=cc.sink, window=cc.window)
try:
    from threadpoolctl import threadpool_info
    blas = [[i.get("internal_api"), i.get("num_threads")] for i in threadpool_info() if i.get("user_api") == "blas"]
except Exception:
    blas = None
for layer, kv, q in calls[: min(4, len(calls))]:  # warm-up (first-call allocations, caches)
    engine.decode_step(q, cache, cc, cfg, layer, kv)
times = []
for rep in range(job["reps"]):
    for layer, kv, q in calls:
        t0 = time.perf_counter()
        engine.decode_step(q, cache, cc, cfg, layer, kv)
        times.append(time.perf_counter() - t0)
print(json.dumps({"backend": doublep.BACKEND, "blas": blas, "times": times}))
"""

# (label, DOUBLEP_KERNELS, BLAS threads: None = all cores)
REF_CONFIGS = (("cython", "cython", None), ("numpy-blas1", "python", 1), ("numpy-blasN", "python", None))


def ref_available():
    return os.path.isdir(os.path.join(REF_DIR, "doublep"))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def ref_decode_times(cache, cc, calls, p1, p2, reps, configs=REF_CONFIGS):
    """Per-call seconds of the reference's decode_step (engine.py:267-278) for
    each backend configuration: {label: {"times": [...], "backend", "blas", "threads"}}."""
    import pickle
    import subprocess
    import tempfile

    with tempfile.NamedTemporaryFile(suffix=".pkl", delete=False) as f:
        pickle.dump({"cache": cache, "cc": cc, "calls": calls, "p1": p1, "p2": p2, "reps": reps}, f)
        job = f.name
    out = {}
    try:
        for label, kern, thr in configs:
            n = str(thr if thr is not None else os.cpu_count())
            env = dict(os.environ, DOUBLEP_KERNELS=kern, OPENBLAS_NUM_THREADS=n, OMP_NUM_THREADS=n,
                       MKL_NUM_THREADS=n)
            r = subprocess.run([sys.executable, "-c", _REF_WORKER, REF_DIR, job], env=env, capture_output=True,
                               text=True, timeout=1800)
            if r.returncode != 0:
                out[label] = {"error": r.stderr.strip().splitlines()[-1:] or ["failed"]}
                continue
            res = json.loads(r.stdout.strip().splitlines()[-1])
            res["threads"] = 1 if kern == "cython" else int(n)  # the Cython kernels never release the GIL
            out[label] = res
    finally:
        os.unlink(job)
    return out


def _ref_import():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import doublep

    return doublep


def ref_cache_from_layer(layer, heads):
    """The reference's KvCache + ClusteredCache (kvcache.py:50, clustering.py:140)
    for kv heads `heads` of a GPU-built single-sequence layer: position-ordered
    f32 keys/values and the device clusters as reference Cluster objects."""
    doublep = _ref_import()
    from doublep.clustering import Cluster, ClusteredCache

    n = layer.n_tokens
    ks, vs, cls = [], [], []
    for h in heads:
        rows_k = layer.keys[0, h, :n].float().cpu().numpy()
        rows_v = layer.values[0, h, :n].float().cpu().numpy()
        perm = layer.perm[0, h, :n].cpu().numpy()
        kp = np.empty_like(rows_k)
        vp = np.empty_like(rows_v)
        kp[perm] = rows_k
        vp[perm] = rows_v
        ks.append(kp)
        vs.append(vp)
        t = layer.head_tables(0, h)
        cls.append([Cluster(members=np.asarray(m, np.int64), centroid=c, size=int(len(m)),
                            value_sum=vm * len(m), value_mean=vm)
                    for m, c, vm in zip(t["members"], t["centroids"], t["value_means"])])
    cache = doublep.KvCache(keys=np.stack(ks)[None], values=np.stack(vs)[None])
    cc = ClusteredCache(source=cache, sink=layer.sink, window=layer.window, clusters=[cls])
    return cache, cc


def summarize_ref(res, scale_up):
    """Pick the fastest configuration; per-step us = median per call x scale_up."""
    rows = {}
    for label, r in res.items():
        if "times" in r:
            med = float(statistics.median(r["times"]))
            rows[label] = {"ms_per_call": med * 1e3, "us_per_step": med * scale_up * 1e6, "calls": len(r["times"]),
                           "backend": r["backend"], "blas": r["blas"], "threads": r["threads"]}
        else:
            rows[label] = r
    ok = {k: v for k, v in rows.items() if "us_per_step" in v}
    best = min(ok, key=lambda k: ok[k]["us_per_step"]) if ok else None
    return best, rows


def run_reference(a):
    """--impl reference: the unmodified reference's decode_step (doublep 0.1.0,
    baseline/_ref) on the host cores, same metric and config, on a bounded
    sample: one kv head of layer 0 generated by the reference's generator
    (workload.py:154-194) and clustered by the reference's own
    build_clustered_cache (NumPy backend, all cores; not timed), then every
    step times decode_step for that head's G q heads under each backend
    configuration; value = the fastest configuration's median per-call time
    x (kv heads x layers x batch x G)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref missing (tools/install_reference.sh)"}))
        return
    os.environ["DOUBLEP_KERNELS"] = "python"  # prefill k-means in this process: NumPy (Cython is ~4x slower)
    doublep = _ref_import()
    from doublep.workload import WorkloadSpec, generate

    n, d, G = a.context, a.head_dim, a.gqa
    spec = WorkloadSpec(context_len=n, head_dim=d, num_kv_heads=1, gqa_group=G, num_layers=1,
                        num_steps=max(a.qsteps, 1), tail_profile=a.profile, seed=0)
    t0 = time.perf_counter()
    cache, trace = generate(spec)
    cc = doublep.build_clustered_cache(cache, sink=4, window=64, seed=0)
    prefill = time.perf_counter() - t0
    steps = a.warmup + a.steps
    calls = [(0, 0, trace.query(s % trace.num_steps, 0, g)) for s in range(steps) for g in range(G)]
    res = ref_decode_times(cache, cc, calls, a.p1, a.p2, reps=1)
    scale_up = a.kv_heads * a.layers * a.batch * G
    best, rows = summarize_ref(res, scale_up)
    val = rows[best]["us_per_step"] if best else None
    line = {
        "impl": "reference", "metric": "decode_us_per_step", "value": val, "unit": "us/step",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": None if val is None else val / 1e3,
        "higher_is_better": False, "scaling": "strong" if a.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (the reference's own generator, host)", "config": workload_config(a, 1),
        "cpu_baseline": {"value": val, "unit": "us/step", "cores": None if best is None else rows[best]["threads"],
                         "kind": "reference", "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                         "backend": best, "configs": rows,
                         "sample": f"doublep 0.1.0 decode_step (unmodified, baseline/_ref) for 1 kv head x {G} q "
                                   f"heads per step at N={n}, {a.warmup}+{a.steps} steps per backend configuration; "
                                   f"median per call x{scale_up} (q heads x layers x batch), labelled extrapolation; "
                                   f"clusters from the reference's build_clustered_cache ({prefill:.1f}s, not timed)"},
        "e2e": {"value": val, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
def _fi_dense(a, layers, qdev, scale, B, hl, G, d, context):
    """The fastest installed dense decode kernel: flashinfer's trtllm-gen
    `trtllm_batch_decode_with_kv_cache` (Blackwell fmhaSm100a cubins; library
    code) over a strided 64-row page view of the same caches (row order does
    not matter to dense attention).  Returns fn(li, s) for graph capture."""
    import torch
    from flashinfer.decode import trtllm_batch_decode_with_kv_cache

    P = 64
    rc = layers[0].row_cap
    if context % P or rc % P:
        raise ValueError("context not a multiple of the page size")
    dev = layers[0].device
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    bt = (torch.arange(B, device=dev)[:, None] * (hl * rc // P) +
          torch.arange(context // P, device=dev)[None]).to(torch.int32)
    sl = torch.full((B,), context, dtype=torch.int32, device=dev)
    npg = B * hl * rc // P - (hl - 1) * rc // P

    def pages(t):
        return torch.as_strided(t, (npg, hl, P, d), (P * d, rc * d, d, 1))

    kv = [(pages(lay.keys), pages(lay.values)) for lay in layers]

    def fn(li, s):
        q = qdev[li][s % a.qsteps]
        return trtllm_batch_decode_with_kv_cache(q, kv[li], ws, bt, sl, context, bmm1_scale=scale)

    return fn


def _measure(a, context, L, dev, world, rank, sampler=None, profile=None, with_dense=True):
    """Build L synthetic layers at `context` (GPU k-means prefill, not timed)
    and time CUDA graphs of the full sparse decode step (plan + attend per
    layer) and of the dense comparator over the same caches."""
    import torch

    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200 import cluster_layer, DecodeWorkspace, ClusteredLayer
    from paper_2602_05191_b200.cache import dtype_code, head_seed
    from paper_2602_05191_b200.workload import generate_layer, generate_queries

    P, r = (a.sim_world, a.sim_rank) if a.sim_world > 1 else (world, rank)
    hl = a.kv_heads // P
    h0 = r * hl
    G, d, B = a.gqa, a.head_dim, a.batch
    lib = N.lib()

    # ---- prefill: synthetic caches + GPU k-means (not timed) -------------
    # Layers are generated and clustered in groups (one batched k-means launch
    # per group, every (layer, sequence, kv head) of the group at once); each
    # group's position-ordered KV is freed as soon as its clustered copy
    # exists, so the resident cache is ONE copy (config 3 at 2 GPUs: 128 GiB
    # per rank) plus one group in flight.  Sequence b of layer li comes from
    # the device generator seeded (layer li, seed b); seeds of the k-means as
    # build_clustered_cache: SeedSequence([0, layer, head]).
    gen_s = prefill_s = 0.0
    per_layer = B * hl * context * d * 2 * 2
    group = max(1, min(L, int(a.prefill_group_gib * (1 << 30)) // max(per_layer, 1)))
    qdev, layers = [], []
    for g0 in range(0, L, group):
        ng = min(group, L - g0)
        t0 = time.perf_counter()
        ks = torch.empty((ng * B, hl, context, d), dtype=torch.bfloat16, device=dev)
        vs = torch.empty_like(ks)
        for li in range(g0, g0 + ng):
            cents = []
            for b in range(B):
                k, v, c = generate_layer(1, a.kv_heads, context, d, layer=li, seed=b, device=dev)
                ks[(li - g0) * B + b] = k[0, h0:h0 + hl]
                vs[(li - g0) * B + b] = v[0, h0:h0 + hl]
                cents.append(c[0, h0:h0 + hl])
                del k, v
            q = generate_queries(np.stack(cents), G, a.qsteps, profile=profile or a.profile, layer=li)
            qdev.append(torch.from_numpy(q).to(dev).to(torch.bfloat16))  # [S,B,Hq,d]
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        seeds = [[head_seed(0, li, h0 + h, b) for h in range(hl)] for li in range(g0, g0 + ng) for b in range(B)]
        big = cluster_layer(ks, vs, fp64_assign=bool(a.fp64_assign), head_seeds=seeds)
        del ks, vs
        torch.cuda.synchronize(dev)
        gen_s += t1 - t0
        prefill_s += time.perf_counter() - t1
        for j in range(ng):  # [ng*B] -> per layer [B]
            sl = lambda t: t[j * B:(j + 1) * B]  # noqa: E731
            lay = ClusteredLayer(sl(big.keys), sl(big.values), sl(big.offs), sl(big.nclusters),
                                 sl(big.centroids), sl(big.value_means), sl(big.perm), big.n_tokens,
                                 big.sink, big.window)
            lay._prefill_k = big._prefill_k
            layers.append(lay)
        del big

    # one workspace reused by every layer, as a serving engine holds it (all
    # layers share the geometry; each plan waits for the previous attention)
    ws0 = DecodeWorkspace(layers[0], G)
    wss = [ws0] * L
    views = [lay.view() for lay in layers]
    scale = 1.0 / math.sqrt(d)

    def layer_step(li, s, stats=None, ev=None):
        ws, v = wss[li], views[li]
        q = qdev[li][s % a.qsteps]
        cs = torch.cuda.current_stream(dev).cuda_stream
        if ev is not None:
            ev[0].record()
        # fused plan: score + two-stage top-p + GQA-union work list (one launch)
        N.check(lib.dp_plan(v, N.ptr(q), dtype_code(q), G, scale, a.p1, a.p2, N.ptr(ws.log_mass), None,
                            N.ptr(ws.counts), N.ptr(ws.stats if stats is None else stats), N.ptr(ws.ws),
                            ws.ws.numel(), cs))
        if ev is not None:
            ev[1].record()
        N.check(lib.dp_attend(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(ws.log_mass), N.ptr(ws.out),
                              N.ptr(ws.lse), N.ptr(ws.ws), ws.ws.numel(), cs))
        if ev is not None:
            ev[2].record()

    def dense_step(li, s, ev=None):
        ws, v = wss[li], views[li]
        q = qdev[li][s % a.qsteps]
        if ev is not None:
            ev[0].record()
        N.check(lib.dp_dense_attention(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(ws.out), N.ptr(ws.lse),
                                       N.ptr(ws.ws), ws.ws.numel(), torch.cuda.current_stream(dev).cuda_stream))
        if ev is not None:
            ev[1].record()

    # ---- stage timing + algorithmic bytes (eager, CUDA events) -----------
    nstage = min(a.qsteps, 4)
    stats_all = torch.zeros((nstage, L, B, hl, 4), dtype=torch.int32, device=dev)
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(L)] for _ in range(nstage)]
    devs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(L)]
    for s in range(nstage):  # warm
        for li in range(L):
            layer_step(li, s, stats_all[s, li])
    torch.cuda.synchronize(dev)
    # park the GPU on a sleep kernel so every launch below is queued before
    # it runs: the events then bracket device time, not host launch gaps
    torch.cuda._sleep(int(2e8))
    for s in range(nstage):
        for li in range(L):
            layer_step(li, s, stats_all[s, li], evs[s][li])
    for li in range(L):
        dense_step(li, 0, devs[li])
    torch.cuda.synchronize(dev)
    stage_ms = np.zeros(2)
    for s in range(nstage):
        for li in range(L):
            e = evs[s][li]
            for j in range(2):
                stage_ms[j] += e[j].elapsed_time(e[j + 1])
    stage_ms /= nstage * L  # per layer
    dense_kernel_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in devs]))
    stats_np = stats_all.cpu().numpy().astype(np.int64)  # [S,L,B,hl,4]
    ncl = np.stack([lay.nclusters.cpu().numpy() for lay in layers]).astype(np.int64)  # [L,B,hl]
    s_kv, s_q, s_o = 2, 2, 4
    Hq_l = hl * G
    qo = B * Hq_l * d * (s_q + s_o)
    U = stats_np[..., 0]
    A = stats_np[..., 1]
    attend_bytes = (U * 2 * d * s_kv + A * d * 4).sum(axis=(2, 3)).mean(axis=0) + qo  # per layer [L]
    score_bytes = (ncl * d * 4 + ncl * 4).sum(axis=(1, 2))  # [L]
    step_bytes = float((attend_bytes + score_bytes).sum())  # all layers, one step
    dense_bytes = float(L * (B * hl * context * 2 * d * s_kv + qo))

    # ---- CUDA graphs of the full step (one per distinct query step) -------
    def capture(fn):
        graphs = []
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for s in range(a.qsteps):
                for li in range(L):
                    fn(li, s)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        for s in range(a.qsteps):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for li in range(L):
                    fn(li, s)
            graphs.append(g)
        return graphs

    def timed(graph_list, steps, warmup, smp=None):
        for s in range(warmup):
            graph_list[s % len(graph_list)].replay()
        torch.cuda.synchronize(dev)
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx = smp if smp is not None else _Null()
        with ctx:
            e0.record()
            for s in range(steps):
                graph_list[s % len(graph_list)].replay()
            e1.record()
            torch.cuda.synchronize(dev)
        barrier(world)
        return e0.elapsed_time(e1) / steps

    graphs = capture(layer_step)
    ms = max_over_ranks(timed(graphs, a.steps, a.warmup, sampler), world, dev)
    del graphs

    # the attention kernel alone, back to back in a graph (PDL-chained as in
    # the step): per-layer workspaces hold each layer's plan
    wsl = [DecodeWorkspace(lay, G) for lay in layers]
    for li in range(L):
        q = qdev[li][0]
        N.check(lib.dp_plan(views[li], N.ptr(q), dtype_code(q), G, scale, a.p1, a.p2, N.ptr(wsl[li].log_mass), None,
                            N.ptr(wsl[li].counts), N.ptr(wsl[li].stats), N.ptr(wsl[li].ws), wsl[li].ws.numel(),
                            torch.cuda.current_stream(dev).cuda_stream))

    def attend_only(li, s):
        w, q = wsl[li], qdev[li][0]
        N.check(lib.dp_attend(views[li], N.ptr(q), dtype_code(q), G, scale, N.ptr(w.log_mass), N.ptr(w.out),
                              N.ptr(w.lse), N.ptr(w.ws), w.ws.numel(), torch.cuda.current_stream(dev).cuda_stream))

    agraphs = capture(attend_only)
    attend_graph_ms = max_over_ranks(timed(agraphs, a.steps, a.warmup), world, dev) / L
    attend_graph_bytes = float((((stats_np[0, :, :, :, 0] * 2 * d * s_kv + stats_np[0, :, :, :, 1] * d * 4)
                                 .sum(axis=(1, 2))) + qo).mean())
    del agraphs, wsl
    dense_ms = fi_ms = None
    fi_note = "skipped"
    if not a.no_dense and with_dense:
        dgraphs = capture(dense_step)
        dense_ms = max_over_ranks(timed(dgraphs, a.steps, a.warmup), world, dev)
        del dgraphs
        if not a.no_fi_dense:
            try:
                fi = _fi_dense(a, layers, qdev, scale, B, hl, G, d, context)
                dense_step(0, 0)
                ref = wss[0].out.clone()
                chk = fi(0, 0).float()
                rel = float((chk - ref).norm() / ref.norm())
                fgraphs = capture(lambda li, s: fi(li, s))
                fi_ms = max_over_ranks(timed(fgraphs, a.steps, a.warmup), world, dev)
                del fgraphs
                fi_note = f"rel-L2 vs dp_dense_attention on layer 0: {rel:.1e}"
            except Exception as e:  # library comparator only; never the product path
                fi_note = f"unavailable: {repr(e)[:160]}"
    return dict(layers=layers, wss=wss, qdev=qdev, ms=ms, dense_ms=dense_ms, fi_ms=fi_ms, fi_note=fi_note,
                stage_ms=stage_ms,
                dense_kernel_ms=dense_kernel_ms, attend_bytes=attend_bytes, step_bytes=step_bytes,
                dense_bytes=dense_bytes, union_frac=float(U.mean() / context), prefill_s=prefill_s, gen_s=gen_s,
                hl=hl, Hq_l=Hq_l, attend_graph_ms=attend_graph_ms, attend_graph_bytes=attend_graph_bytes)


def run_b200(a):
    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2602_05191_b200 import DecodeGraph, sparse_attention

    if a.kv_heads % world:
        raise SystemExit(f"kv heads {a.kv_heads} not divisible by {world} ranks")
    G, d, L, B = a.gqa, a.head_dim, a.layers, a.batch
    sampler = ClockSampler(local)
    res = _measure(a, a.context, L, dev, world, rank, sampler)
    clocks = sampler.summary()
    layers, wss, qdev, ms, dense_ms = res["layers"], res["wss"], res["qdev"], res["ms"], res["dense_ms"]
    hl, Hq_l = res["hl"], res["Hq_l"]
    stage_ms, attend_bytes = res["stage_ms"], res["attend_bytes"]
    step_bytes, dense_bytes, union_frac = res["step_bytes"], res["dense_bytes"], res["union_frac"]
    prefill_s, gen_s = res["prefill_s"], res["gen_s"]
    attend_ms = stage_ms[1]
    attend_gbs = float(attend_bytes.mean() / (attend_ms * 1e-3) / 1e9)
    res_attend_graph_ms, res_attend_graph_bytes = res["attend_graph_ms"], res["attend_graph_bytes"]

    # ---- e2e through the public API with host buffers ---------------------
    e2e = None
    if not a.no_e2e:
        # the step's inputs (every layer's q) come from pinned host memory in one
        # copy; every layer's output lands in one device buffer read back once
        qh = torch.empty((a.qsteps, L, B, Hq_l, d), dtype=torch.bfloat16).pin_memory()
        for li in range(L):
            qh[:, li].copy_(qdev[li].cpu())
        oh = torch.empty((L, B, Hq_l, d), dtype=torch.float32).pin_memory()
        qd = torch.empty((L, B, Hq_l, d), dtype=torch.bfloat16, device=dev)
        od = torch.empty((L, B, Hq_l, d), dtype=torch.float32, device=dev)

        def e2e_eager(s):
            qd.copy_(qh[s % a.qsteps], non_blocking=True)
            for li in range(L):
                sparse_attention(qd[li], layers[li], a.p1, a.p2, workspace=wss[li], out=od[li])
            oh.copy_(od, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()

        # the serving form of the same API: the 32 per-layer calls captured once
        # (DecodeGraph) with the pinned copies inside the graph -- one graph per
        # distinct query step (each reads its own pinned slice), replayed per step
        qd.copy_(qh[0])  # real queries in the graph's input buffer before its eager warm-up
        graphs = [DecodeGraph(layers, qd, a.p1, a.p2, out=od, workspace=wss[0], host_q=qh[s], host_out=oh)
                  for s in range(a.qsteps)]

        def e2e_graph(s):
            graphs[s % a.qsteps].replay()
            torch.cuda.current_stream(dev).synchronize()

        def timed_e2e(fn):
            for s in range(a.warmup):
                fn(s)
            barrier(world)
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in range(a.steps):
                fn(s)
            e1.record()
            torch.cuda.synchronize(dev)
            wall = (time.perf_counter() - t0) / a.steps * 1e3
            return max_over_ranks(max(e0.elapsed_time(e1) / a.steps, wall), world, dev)

        e2e_ms = timed_e2e(e2e_graph)
        eager_ms = timed_e2e(e2e_eager)
        e2e = {"value": e2e_ms * 1e3, "unit": "us/step", "h2d_bytes_per_step": int(L * B * Hq_l * d * 2),
               "d2h_bytes_per_step": int(L * B * Hq_l * d * 4),
               "path": "paper_2602_05191_b200.DecodeGraph (the step's 32 sparse_attention calls and the pinned "
                       "host copies captured once as a CUDA graph, one shared workspace), replayed per step: all "
                       "layers' q in from pinned host memory (layer 0 first, the rest overlapping it), every "
                       "layer's output back to pinned host memory as soon as it is ready, host sync per step",
               "eager_us_per_step": eager_ms * 1e3,
               "eager_path": "paper_2602_05191_b200.sparse_attention per layer, eager, same copies"}

    # ---- CPU baseline (rank 0, N=1 only): the reference's own decode_step --
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and ref_available():
        nh = min(a.cpu_sample_heads, hl)
        rcache, rcc = ref_cache_from_layer(layers[0], range(nh))
        qs = qdev[0][:4, 0].float().cpu().numpy()  # [4 steps, Hq, d]
        calls = [(0, h, qs[s, h * G + g]) for s in range(qs.shape[0]) for h in range(nh) for g in range(G)]
        res_ref = ref_decode_times(rcache, rcc, calls, a.p1, a.p2, reps=1,
                                   configs=(REF_CONFIGS[0], REF_CONFIGS[2]))
        scale_up = a.kv_heads * G * L * B
        best, rows = summarize_ref(res_ref, scale_up)
        if best is not None:
            cpu = {"value": rows[best]["us_per_step"], "unit": "us/step", "cores": rows[best]["threads"],
                   "kind": "reference", "cpu_model": cpu_model(), "host_cores": os.cpu_count(), "backend": best,
                   "configs": rows,
                   "sample": f"doublep 0.1.0 decode_step (unmodified, baseline/_ref) on layer 0, {nh} kv heads x "
                             f"{G} q heads x 4 query steps of the GPU-built clusters (as reference Cluster objects); "
                             f"median {rows[best]['ms_per_call']:.2f} ms per q-head-step, labelled extrapolation "
                             f"x{scale_up} (all q heads, layers, batch)"}

    fi_ms, fi_note = res["fi_ms"], res["fi_note"]
    # ---- the 'mixed' stress profile (workload.py:83-89) at the same context --
    mixed = None
    del layers, wss, qdev, res
    torch.cuda.empty_cache()
    if a.mixed_layers and a.profile != "mixed":
        rm = _measure(a, a.context, a.mixed_layers, dev, world, rank, profile="mixed")
        mixed = {"profile": "mixed", "context": a.context, "layers_timed": a.mixed_layers,
                 "us_per_layer": rm["ms"] * 1e3 / a.mixed_layers,
                 "us_per_step_32_layers": rm["ms"] * 1e3 / a.mixed_layers * 32,
                 "dense_us_per_layer": None if rm["dense_ms"] is None else rm["dense_ms"] * 1e3 / a.mixed_layers,
                 "fi_dense_us_per_layer": None if rm["fi_ms"] is None else rm["fi_ms"] * 1e3 / a.mixed_layers,
                 "union_exact_rows_frac": rm["union_frac"],
                 "stage_us_per_layer": {"plan": rm["stage_ms"][0] * 1e3, "attend": rm["stage_ms"][1] * 1e3},
                 "attend_gbs": float(rm["attend_bytes"].mean() / (rm["stage_ms"][1] * 1e-3) / 1e9)}
        dm = [x for x in (rm["dense_ms"], rm["fi_ms"]) if x is not None]
        mixed["speedup_vs_fastest_dense"] = min(dm) / rm["ms"] if dm else None
        del rm
        torch.cuda.empty_cache()

    # ---- secondary workload: the same step at 128K context (fewer layers) --
    long_ctx = None
    if a.long_context and a.long_context != a.context:
        r2 = _measure(a, a.long_context, a.long_layers, dev, world, rank)
        a_ms = r2["stage_ms"][1]
        long_ctx = {
            "context": a.long_context, "layers_timed": a.long_layers,
            "us_per_layer": r2["ms"] * 1e3 / a.long_layers,
            "us_per_step_32_layers": r2["ms"] * 1e3 / a.long_layers * 32,
            "dense_us_per_layer": None if r2["dense_ms"] is None else r2["dense_ms"] * 1e3 / a.long_layers,
            "fi_dense_us_per_layer": None if r2["fi_ms"] is None else r2["fi_ms"] * 1e3 / a.long_layers,
            "speedup_vs_dense": None if r2["dense_ms"] is None else
            min(x for x in (r2["dense_ms"], r2["fi_ms"]) if x is not None) / r2["ms"],
            "speedup_vs": "the fastest of dp_dense_attention and flashinfer trtllm-gen",
            "stage_us_per_layer": {"plan": r2["stage_ms"][0] * 1e3, "attend": a_ms * 1e3},
            "attend_algorithmic_bytes": float(r2["attend_bytes"].mean()),
            "attend_gbs": float(r2["attend_bytes"].mean() / (a_ms * 1e-3) / 1e9),
            "dense_kernel_gbs": r2["dense_bytes"] / a.long_layers / (r2["dense_kernel_ms"] * 1e-3) / 1e9,
            "union_exact_rows_frac": r2["union_frac"],
            "attend_in_graph": {"us_per_launch": r2["attend_graph_ms"] * 1e3,
                                "gbs": r2["attend_graph_bytes"] / (r2["attend_graph_ms"] * 1e-3) / 1e9},
        }

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None  # ncu-measured DRAM bytes per attention launch, when profiled at this workload
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if a.context == 32768 and a.batch == 1 and a.gqa == 4 and a.kv_heads == 8 and world == 1:
            traffic = float(tj["attn_tc_kernel_sparse_32k_b1_g4"])
    except Exception:
        pass
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    launches = a.steps * L * 2  # plan_kernel (score+select+worklist), attn_tc_kernel (+ fused merge)
    if rank == 0:
        line = {
            "metric": "decode_us_per_step", "value": ms * 1e3, "unit": "us/step", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference blob law on device, Philox); random-init caches, no checkpoint",
            "config": workload_config(a, world),
            "roofline": {"bound": "hbm", "achieved": attend_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": attend_gbs / hbm_peak, "frac_vs_8tbs": attend_gbs / 8000.0, "traffic": traffic,
                         "traffic_source": "profiles/traffic.json (ncu --set full, dram read+write per launch)",
                         "kernel": "dp_attend = attn_tc_kernel (gathered split-KV attention + fused LSE merge), one launch per layer",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": float(attend_bytes.mean())},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "stage_us_per_layer": {"plan": stage_ms[0] * 1e3, "attend": stage_ms[1] * 1e3},
            "attend_in_graph": {"us_per_launch": res_attend_graph_ms * 1e3,
                                "algorithmic_bytes_per_launch": res_attend_graph_bytes,
                                "gbs": res_attend_graph_bytes / (res_attend_graph_ms * 1e-3) / 1e9,
                                "frac": res_attend_graph_bytes / (res_attend_graph_ms * 1e-3) / 1e9 / hbm_peak,
                                "note": "attn_tc_kernel launches back to back in a CUDA graph (PDL-chained), per-layer "
                                        "work lists from one plan each; the roofline object above times each launch "
                                        "between CUDA events (no PDL overlap)"},
            "step_algorithmic_bytes": step_bytes,
            "step_roofline_frac": step_bytes / (ms * 1e-3) / 1e9 / hbm_peak,
            "union_exact_rows_frac": union_frac,
            "dense_us_per_step": None if dense_ms is None else min(x for x in (dense_ms, fi_ms) if x is not None) * 1e3,
            "dense_comparators_us_per_step": {
                "dp_dense_attention": None if dense_ms is None else dense_ms * 1e3,
                "flashinfer_trtllm_gen": None if fi_ms is None else fi_ms * 1e3,
                "flashinfer_note": fi_note},
            "dense_roofline_frac": None if dense_ms is None else dense_bytes / (dense_ms * 1e-3) / 1e9 / hbm_peak,
            "speedup_vs_dense": None if dense_ms is None else min(x for x in (dense_ms, fi_ms) if x is not None) / ms,
            "speedup_vs": "the fastest dense kernel measured in this run (dp_dense_attention, flashinfer trtllm-gen)",
            "mixed_profile": mixed,
            "prefill_s": prefill_s, "generate_s": gen_s,
            "long_context": long_ctx,
        }
        line["attend_in_graph"]["frac_vs_8tbs"] = line["attend_in_graph"]["gbs"] / 8000.0
        if long_ctx is not None:
            long_ctx["attend_roofline_frac"] = long_ctx["attend_gbs"] / hbm_peak
            long_ctx["attend_in_graph"]["frac"] = long_ctx["attend_in_graph"]["gbs"] / hbm_peak
            long_ctx["attend_in_graph"]["frac_vs_8tbs"] = long_ctx["attend_in_graph"]["gbs"] / 8000.0
            long_ctx["dense_kernel_roofline_frac"] = long_ctx["dense_kernel_gbs"] / hbm_peak
        print(json.dumps(line), flush=True)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def measured_peak():
    """(HBM GB/s, source): MEASURED_PEAKS.json (driver-written) or the
    profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        peaks = {}
    return float(peaks.get("hbm_gbs", 6650.0)), ("measured" if "hbm_gbs" in peaks else "fallback")


def run_seqshard(a):
    """Config 5: 1M-token single-sequence decode, sequence-sharded over P GPUs
    with the reference's global selection (paper_2602_05191_b200.seqshard):
    per layer each rank scores its slice of the cluster table, the log-mass
    slices are all-gathered, dp_select_global runs the two-stage top-p over
    the whole table, the rank attends over its exact clusters / pseudo-rows
    and the partials are all-gathered and merged (dp_lse_merge).  Caches: each
    rank clusters its own 1/P of the tokens into 1/P of the clusters (the
    cluster-partitioned layout; the GLOBAL k-means of seqshard.shard_cluster_layer
    is ~32K sequential all-reduce rounds at 1M and is exercised by the tests,
    not here).  Without torchrun the other ranks' slices are stand-ins (this
    rank's own slice repeated) and the collectives are not timed."""
    import torch

    from paper_2602_05191_b200 import _native as N
    from paper_2602_05191_b200 import cluster_layer
    from paper_2602_05191_b200.cache import dtype_code, head_seed
    import torch.distributed as dist

    from paper_2602_05191_b200.seqshard import Comm
    from paper_2602_05191_b200.sharding import seq_shard_bounds
    from paper_2602_05191_b200.workload import generate_layer, generate_queries

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    P = a.seq_shards
    real = world > 1
    if real and world != P:
        raise SystemExit(f"--seq-shards {P} needs {P} ranks (got {world})")
    r = rank if real else a.sim_rank
    comm = Comm() if real else None
    L, G, d, H = a.layers, a.gqa, a.head_dim, a.kv_heads
    Hq = H * G
    lo, hi = seq_shard_bounds(a.context, P, r)
    n_r = hi - lo
    sink = 4 if r == 0 else 0
    window = 64 if r == P - 1 else 0
    lib = N.lib()
    t0 = time.perf_counter()
    layers, qs = [], []
    for li in range(L):
        k, v, c = generate_layer(1, H, n_r, d, layer=li, seed=1000 + r, device=dev)
        seeds = [[head_seed(0, li, h, 1000 + r) for h in range(H)]]
        lay = cluster_layer(k, v, sink=sink, window=window, head_seeds=seeds)
        del k, v
        layers.append(lay)
        qs.append(torch.from_numpy(generate_queries(c, G, a.qsteps, profile=a.profile, layer=li)).to(dev)
                  .to(torch.bfloat16))  # [S, 1, Hq, d]
    torch.cuda.synchronize(dev)
    prefill_s = time.perf_counter() - t0
    cap = max(lay.cluster_cap for lay in layers)
    ld = P * cap
    scale = 1.0 / math.sqrt(d)
    lm = torch.zeros((1, Hq, cap), dtype=torch.float64, device=dev)
    st = torch.zeros((1, Hq, cap), dtype=torch.uint8, device=dev)
    g_lm = torch.full((Hq, ld), -math.inf, dtype=torch.float64, device=dev)
    g_st = torch.zeros((Hq, ld), dtype=torch.uint8, device=dev)
    g_cnt = torch.zeros((Hq, 2), dtype=torch.int32, device=dev)
    g_k = torch.full((Hq,), ld, dtype=torch.int32, device=dev)
    g_ws = torch.empty((lib.dp_select_global_workspace_bytes(Hq, ld),), dtype=torch.uint8, device=dev)
    out = torch.zeros((1, Hq, d), dtype=torch.float32, device=dev)
    lse = torch.zeros((1, Hq), dtype=torch.float32, device=dev)
    parts_o = torch.zeros((P, 1, Hq, d), dtype=torch.float32, device=dev)
    parts_l = torch.zeros((P, 1, Hq), dtype=torch.float32, device=dev)
    merged = torch.zeros_like(out)
    merged_l = torch.zeros_like(lse)
    wsb = max(lib.dp_decode_workspace_bytes(lay.view(), G) for lay in layers)
    ws = torch.zeros((wsb,), dtype=torch.uint8, device=dev)
    views = [lay.view() for lay in layers]
    stats = torch.zeros((L, 1, H, 4), dtype=torch.int32, device=dev)
    # dp_plan's shape limit; the in-place selection's (P * cap <= 65536)
    use_plan = cap <= 4096 and P * cap <= 65536 and os.environ.get("DP_SEQ_UNFUSED") is None
    parts_lm = torch.full((P, Hq, cap), -math.inf, dtype=torch.float64, device=dev)
    h_st = torch.zeros((Hq, P * cap), dtype=torch.uint8, device=dev)
    h_k = torch.full((Hq,), P * cap, dtype=torch.int32, device=dev)

    def layer_step(li, s, ev=None):
        cs = torch.cuda.current_stream(dev).cuda_stream
        q = qs[li][s % a.qsteps]
        lay, v = layers[li], views[li]
        if ev is not None:
            ev[0].record()
        if use_plan:  # the fused plan's scoring phase (-inf past K); its work-list phase runs on the global states below
            N.check(lib.dp_plan_score(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(lm), N.ptr(ws), ws.numel(), cs))
        else:
            lm.fill_(-math.inf)
            N.check(lib.dp_score(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(lm), cs))
        if ev is not None:
            ev[1].record()
        if use_plan:  # in place: the selection reads the gathered [P, Hq, cap] slices, the plan its slice of states
            if real:
                dist.all_gather_into_tensor(parts_lm, lm[0])
            else:  # stand-ins for the other ranks' slices: this rank's own slice
                parts_lm.copy_(lm[0].unsqueeze(0).expand(P, Hq, cap))
            if ev is not None:
                ev[2].record()
            N.check(lib.dp_select_global_parts(N.ptr(parts_lm), Hq, P, cap, N.ptr(h_k), a.p1, a.p2, N.ptr(h_st),
                                               N.ptr(g_cnt), N.ptr(g_ws), g_ws.numel(), cs))
            if ev is not None:
                ev[3].record()
            N.check(lib.dp_plan_given(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(lm), N.ptr(h_st[:, r * cap:]),
                                      P * cap, N.ptr(stats[li]), N.ptr(ws), ws.numel(), cs))
            N.check(lib.dp_attend(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(lm), N.ptr(out), N.ptr(lse), N.ptr(ws),
                                  ws.numel(), cs))
            if ev is not None:
                ev[4].record()
            merge_step()
            if ev is not None:
                ev[5].record()
            return
        if real:
            g_lm.view(Hq, P, cap).copy_(comm.all_gather(lm[0]).permute(1, 0, 2))
        else:  # stand-ins for the other ranks' slices: this rank's own slice
            g_lm.view(Hq, P, cap).copy_(lm[0].unsqueeze(1).expand(Hq, P, cap))
        if ev is not None:
            ev[2].record()
        N.check(lib.dp_select_global(N.ptr(g_lm), Hq, ld, N.ptr(g_k), a.p1, a.p2, N.ptr(g_st), N.ptr(g_cnt),
                                     N.ptr(g_ws), g_ws.numel(), cs))
        st[0].copy_(g_st.view(Hq, P, cap)[:, r])
        if ev is not None:
            ev[3].record()
        N.check(lib.dp_sparse_attention(v, N.ptr(q), dtype_code(q), G, scale, N.ptr(lm), N.ptr(st), N.ptr(out),
                                        N.ptr(lse), N.ptr(stats[li]), N.ptr(ws), ws.numel(), cs))
        if ev is not None:
            ev[4].record()
        merge_step()
        if ev is not None:
            ev[5].record()

    def merge_step():
        cs = torch.cuda.current_stream(dev).cuda_stream
        if real:
            dist.all_gather_into_tensor(parts_o, out)
            dist.all_gather_into_tensor(parts_l, lse)
        else:
            parts_o.copy_(out.unsqueeze(0).expand_as(parts_o))
            parts_l.copy_(lse.unsqueeze(0).expand_as(parts_l))
        N.check(lib.dp_lse_merge(N.ptr(parts_o), N.ptr(parts_l), P, Hq, d, N.ptr(merged), N.ptr(merged_l), cs))

    sampler = ClockSampler(local)
    for s in range(a.warmup):
        for li in range(L):
            layer_step(li, s)
    torch.cuda.synchronize(dev)
    if os.environ.get("DP_DUMP_GLM"):  # tools/gsel_probe.py: the last layer's global log-mass table
        torch.save(g_lm.cpu(), os.environ["DP_DUMP_GLM"])
    graphs = None
    if not real:  # one CUDA graph per distinct query step (the collectives of a real run stay eager)
        graphs = []
        for s in range(a.qsteps):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for li in range(L):
                    layer_step(li, s)
            graphs.append(g)
        for s in range(a.warmup):
            graphs[s % len(graphs)].replay()
        torch.cuda.synchronize(dev)
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record()
        for s in range(a.steps):
            if graphs is not None:
                graphs[s % len(graphs)].replay()
            else:
                for li in range(L):
                    layer_step(li, s)
        e1.record()
        torch.cuda.synchronize(dev)
    barrier(world)
    del graphs
    ms = max_over_ranks(e0.elapsed_time(e1) / a.steps, world, dev)
    # stage split (eager, CUDA events): score / gather / select / attend / merge
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(L)]
    torch.cuda._sleep(int(1e8))
    for li in range(L):
        layer_step(li, 0, evs[li])
    torch.cuda.synchronize(dev)
    stage = np.mean([[e[j].elapsed_time(e[j + 1]) for j in range(5)] for e in evs], axis=0) * 1e3
    st_np = stats.cpu().numpy().astype(np.int64)
    U, A = st_np[..., 0], st_np[..., 1]
    ncl = np.stack([lay.nclusters.cpu().numpy() for lay in layers]).astype(np.int64)
    attend_bytes = (U * 2 * d * 2 + A * d * 4).sum(axis=(1, 2)) + Hq * d * (2 + 4)  # [L]
    step_bytes = float(attend_bytes.sum() + (ncl * (d * 4 + 4)).sum())
    dense_bytes = float(L * H * n_r * 2 * d * 2)
    hbm_peak, peak_src = measured_peak()
    if rank == 0:
        line = {
            "metric": "decode_us_per_step", "value": ms * 1e3, "unit": "us/step", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference blob law on device, Philox); random-init caches, no checkpoint",
            "config": {"workload": f"doublep-decode llama-3.1-8b-shape L{L} B1 N{a.context} Hq{Hq}/Hkv{H} d{d} bf16 "
                                   f"p=({a.p1},{a.p2}) {a.profile} sequence-sharded P={P}",
                       "layers": L, "context": a.context, "seq_shards": P, "rank_tokens": n_r,
                       "parallelism": (f"sequence shards over {P} GPUs" if real else
                                       f"sequence shard {r}/{P} measured alone on one GPU (collectives not timed; "
                                       f"other ranks' log-mass slices and partials are stand-ins)"),
                       "global_clusters": int(P * ncl.sum(axis=(1, 2)).mean() / H),
                       "caches": "each rank clusters its own 1/P of the tokens (cluster-partitioned layout)",
                       "l2": "inputs larger than L2 (each layer's KV > 126 MB; layers cycled)"},
            "stage_us_per_layer": {"score": stage[0], "gather": stage[1], "select_global": stage[2],
                                   "attend": stage[3], "merge": stage[4]},
            "attend_roofline": {"bound": "hbm", "achieved": float(attend_bytes.mean() / (stage[3] * 1e-6) / 1e9),
                                "peak": hbm_peak, "unit": "GB/s", "peak_source": peak_src},
            "step_algorithmic_bytes": step_bytes, "dense_bytes_per_rank": dense_bytes,
            "union_exact_rows_frac": float(U.mean() / n_r),
            "collective_bytes_per_layer": {"all_gather_log_mass": Hq * ld * 8, "all_gather_partials": P * Hq * (d + 1) * 4},
            "prefill_s": prefill_s, "clocks": sampler.summary(),
            "timing": "CUDA graph of the L-layer step" if not real else "eager (NCCL collectives in the step)",
            "gpu_launches": L * a.steps * 7,
        }
        print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.seq_shards > 1:
        run_seqshard(a)
    else:
        run_b200(a)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
