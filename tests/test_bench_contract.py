"""bench.py contract on CPU: the reference arm runs at a tiny size and prints
one JSON line with the keys the driver reads."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--context", "1024",
                        "--layers", "2", "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    if "unavailable" in d:  # baseline/_ref not installed (tools/install_reference.sh)
        assert not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "doublep"))
        return
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["higher_is_better"] is False and d["value"] > 0
    cb = d["cpu_baseline"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and cb["kind"] == "reference" and cb["value"] == d["value"]
    assert set(cb["configs"]) == {"cython", "numpy-blas1", "numpy-blasN"} and cb["backend"] in cb["configs"]
    assert cb["cores"] >= 1 and "workload" in d["config"]
