"""Route the reference package's operator API to this package.

This is the maintainer-side switch of INTEGRATION.md §1(a), packaged as a
function so the same wiring can be applied to an installed ``doublep`` (the
reference, /root/reference/pkg) without editing its sources:

    import doublep
    from paper_2602_05191_b200 import integration
    handle = integration.install(doublep)     # doublep.* now runs on the B200 path
    ...
    handle.uninstall()

``install`` rebinds, in the reference modules, every operator that takes a
cache, a clustered cache or a plan (engine.py:122-370, clustering.py:266,
metrics.py:26-76) plus the names other reference modules imported from
them (cli.py:31 ``build_clustered_cache``, the package's top-level
re-exports).  The reference's own objects keep working: its ``KvCache``
(numpy) is copied to the device once, a ``ClusteredCache`` built by the
reference's CPU k-means is uploaded once into the device layout, its
``DoublePConfig`` is read by attribute.  Attention outputs come back as the
reference's ``AttentionOutput`` class so ``metrics.output_error``'s
isinstance check (metrics.py:18-19) behaves as before.

Doing it at import time instead (the snippet in INTEGRATION.md, placed at the
end of ``doublep/engine.py`` and ``doublep/clustering.py`` under
``DOUBLEP_KERNELS=b200``) binds the same functions.
"""

from __future__ import annotations

import importlib
import sys

from . import cache as _cache
from . import engine as _engine
from . import metrics as _metrics

# reference module -> {name: replacement factory(ref_modules) -> callable}
_ENGINE_FUNCS = (
    "estimate_cluster_distribution", "plan_selection", "sparse_attention", "decode_step", "full_attention",
    "full_attention_weights", "true_token_weights", "baseline_token_topk", "baseline_cluster_topk",
    "baseline_token_topp_fixed_budget", "build_cache_for_config", "build_clustered_cache",
)
_METRICS_FUNCS = ("recovered_mass", "adaptive_token_budget", "cluster_approx_error")


class Handle:
    """Undo record of one ``install``."""

    def __init__(self):
        self._saved = []

    def _set(self, mod, name, value):
        self._saved.append((mod, name, getattr(mod, name)))
        setattr(mod, name, value)

    def uninstall(self):
        for mod, name, value in reversed(self._saved):
            setattr(mod, name, value)
        self._saved.clear()

    def original(self, qualname):
        """The function a rebound name held before install ("doublep.engine.decode_step")."""
        mod, _, name = qualname.rpartition(".")
        for m, n, v in self._saved:
            if m.__name__ == mod and n == name:
                return v
        raise KeyError(qualname)

    @property
    def patched(self):
        return [f"{m.__name__}.{n}" for m, n, _ in self._saved]


def _modules(pkg):
    name = pkg.__name__ if pkg is not None else "doublep"
    base = pkg if pkg is not None else importlib.import_module(name)
    mods = {"pkg": base}
    for sub in ("engine", "clustering", "metrics", "cli"):
        mods[sub] = importlib.import_module(f"{name}.{sub}")
    return mods


def install(pkg=None):
    """Bind the reference package ``pkg`` (default: ``import doublep``) to the
    B200 operators.  Returns a Handle whose ``uninstall()`` restores it."""
    mods = _modules(pkg)
    ref_engine = mods["engine"]
    RefOut = ref_engine.AttentionOutput

    def as_ref(o):
        return RefOut(output=o.output, normalizer=o.normalizer, exact_token_count=o.exact_token_count,
                      approx_cluster_count=o.approx_cluster_count)

    def sparse_attention(q, cache, cc, plan, layer, kv_head):
        return as_ref(_engine.sparse_attention(q, cache, cc, plan, layer, kv_head))

    def decode_step(q, cache, cc, cfg, layer, kv_head):
        out, plan, est = _engine.decode_step(q, cache, cc, cfg, layer, kv_head)
        return as_ref(out), plan, est

    def full_attention(q, cache, layer, kv_head):
        return as_ref(_engine.full_attention(q, cache, layer, kv_head))

    def baseline_token_topk(q, cache, budget, layer, kv_head):
        out, captured = _metrics.baseline_token_topk(q, cache, budget, layer, kv_head)
        return as_ref(out), captured

    def baseline_cluster_topk(q, cache, cc, budget, layer, kv_head):
        return as_ref(_metrics.baseline_cluster_topk(q, cache, cc, budget, layer, kv_head))

    def baseline_token_topp_fixed_budget(q, cache, est_budget, p, layer, kv_head):
        out, rec = _metrics.baseline_token_topp_fixed_budget(q, cache, est_budget, p, layer, kv_head)
        return as_ref(out), rec

    repl = {
        "estimate_cluster_distribution": _engine.estimate_cluster_distribution,
        "plan_selection": _engine.plan_selection,
        "sparse_attention": sparse_attention,
        "decode_step": decode_step,
        "full_attention": full_attention,
        "full_attention_weights": _metrics.full_attention_weights,
        "true_token_weights": _metrics.true_token_weights,
        "baseline_token_topk": baseline_token_topk,
        "baseline_cluster_topk": baseline_cluster_topk,
        "baseline_token_topp_fixed_budget": baseline_token_topp_fixed_budget,
        "build_cache_for_config": _engine.build_cache_for_config,
        "build_clustered_cache": _cache.build_clustered_cache,
        "recovered_mass": _metrics.recovered_mass,
        "adaptive_token_budget": _metrics.adaptive_token_budget,
        "cluster_approx_error": _metrics.cluster_approx_error,
    }
    h = Handle()
    for name in _ENGINE_FUNCS:
        h._set(ref_engine, name, repl[name])
    h._set(mods["clustering"], "build_clustered_cache", repl["build_clustered_cache"])
    for name in _METRICS_FUNCS:
        h._set(mods["metrics"], name, repl[name])
    h._set(mods["cli"], "build_clustered_cache", repl["build_clustered_cache"])
    for name in _ENGINE_FUNCS + _METRICS_FUNCS:  # top-level re-exports (doublep/__init__.py)
        if hasattr(mods["pkg"], name):
            h._set(mods["pkg"], name, repl[name])
    # modules that already did `from doublep.engine import X` (e.g. a test
    # module imported before install) keep their binding; rebind those too
    originals = {id(v): n for m, n, v in h._saved}
    for mod in list(sys.modules.values()):
        d = getattr(mod, "__dict__", None)
        if not d or mod in mods.values() or getattr(mod, "__name__", "").startswith(__package__):
            continue
        for k, v in list(d.items()):
            n = originals.get(id(v))
            if n is not None and k == n:
                h._set(mod, k, repl[n])
    return h


def install_kernels(pkg=None):
    """Make ``paper_2602_05191_b200.kernels`` the reference's kernel backend:
    the one-level-lower binding (the reference's own plugin seam,
    kernels.py:17-29) -- every ``kernels.X`` call the reference makes
    (engine.py:128-361, clustering.py:85, numerics.py:35-44,
    selection.py:82) then runs on the GPU through dp_kn_*.  ``BACKEND`` reads
    "b200".  Returns a Handle whose ``uninstall()`` restores the previous
    backend."""
    from . import kernels as b200_kernels

    name = pkg.__name__ if pkg is not None else "doublep"
    base = pkg if pkg is not None else importlib.import_module(name)
    ref_kernels = importlib.import_module(f"{name}.kernels")
    h = Handle()
    h._set(ref_kernels, "_impl", b200_kernels)
    h._set(ref_kernels, "BACKEND", b200_kernels.BACKEND)
    if hasattr(base, "BACKEND"):
        h._set(base, "BACKEND", b200_kernels.BACKEND)
    return h
