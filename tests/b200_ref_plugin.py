"""pytest plugin: run the reference's own test suite with the reference's
operator API bound to the B200 path (paper_2602_05191_b200.integration).

    PYTHONPATH=baseline/_ref:.:tests python -m pytest -p b200_ref_plugin baseline/_ref/tests/test_engine.py

B200_REF_BIND selects what is bound: "ops" (default; the operator API,
integration.install) or "kernels" (the reference's kernel plugin seam,
integration.install_kernels: every kernels.X call on the GPU, the reference's
engine and clustering unchanged above it).

Loaded before any conftest, so the reference's conftest and test modules
import the rebound functions."""

import json
import os

_calls = {}


class _CountingKernels:
    """The B200 kernels module, counting calls per name (so a caller can see
    the seam was actually exercised)."""

    def __init__(self, mod):
        self._mod = mod

    def __getattr__(self, name):
        f = getattr(self._mod, name)
        if not callable(f):
            return f

        def wrapped(*a, **k):
            _calls[name] = _calls.get(name, 0) + 1
            return f(*a, **k)

        return wrapped


def pytest_configure(config):
    import doublep

    from paper_2602_05191_b200 import integration

    mode = os.environ.get("B200_REF_BIND", "ops")
    if mode == "kernels":
        from paper_2602_05191_b200 import kernels

        config._b200_handle = integration.install_kernels(doublep)
        doublep.kernels._impl = _CountingKernels(kernels)
    else:
        config._b200_handle = integration.install(doublep)
    config._b200_mode = mode


def pytest_unconfigure(config):
    path = os.environ.get("B200_REF_SEAM_COUNTS")
    if path and getattr(config, "_b200_mode", None) == "kernels":
        with open(path, "w") as f:
            json.dump(_calls, f)


def pytest_report_header(config):
    h = getattr(config, "_b200_handle", None)
    return (f"doublep {getattr(config, '_b200_mode', 'ops')} bound to paper_2602_05191_b200 "
            f"({len(h.patched) if h else 0} names)")
