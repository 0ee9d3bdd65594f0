"""pytest plugin: run the reference's own test suite with the reference's
operator API bound to the B200 path (paper_2602_05191_b200.integration).

    PYTHONPATH=baseline/_ref:.:tests python -m pytest -p b200_ref_plugin baseline/_ref/tests/test_engine.py

Loaded before any conftest, so the reference's conftest and test modules
import the rebound functions."""


def pytest_configure(config):
    import doublep

    from paper_2602_05191_b200 import integration

    config._b200_handle = integration.install(doublep)


def pytest_report_header(config):
    h = getattr(config, "_b200_handle", None)
    return f"doublep operators bound to paper_2602_05191_b200 ({len(h.patched) if h else 0} names)"
