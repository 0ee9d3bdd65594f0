"""Golden pyexport dumps written by the REAL reference exporter (test infrastructure).

    python oracle/gen_golden_pyexport.py      # in the build container (/root/reference present)

Runs the reference's pyexport.exporter.export (pkg/pyexport/src/pyexport/
exporter.py:107-175) on its download-free synthetic-llama for a fixed prompt
in float32 and float16 and stores the DPKV files and manifests under
tests/golden/, so tests/test_capture.py can check paper_2602_05191_b200.capture
byte for byte without /root/reference at run time.
"""
import json
import os
import sys

os.environ["DOUBLEP_KERNELS"] = "python"
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/pyexport/src")

from pyexport.exporter import export  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
PROMPT = ("The export path is exercised with a prompt long enough to give the attention maps some structure: "
          "repeated phrases, punctuation, and a little variation.")
STEPS = 6


def main():
    for dtype in ("float32", "float16"):
        path = os.path.join(OUT, f"pyexport_synth_{dtype}.dpkv")
        man = export("synthetic-llama", PROMPT, STEPS, path, dtype=dtype, seed=0, prompt_source="golden")
        with open(path + ".manifest.json") as f:
            assert json.load(f) == man.to_dict()
        print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
