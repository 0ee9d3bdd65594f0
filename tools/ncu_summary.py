"""Summarise an ncu launch list (--metrics gpu__time_duration.sum) and a
--set full report into markdown for profiles/.

    python tools/ncu_summary.py launches.csv report.ncu-rep > profiles/x.md
"""
import collections
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "")
            scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
            agg[name].append(float(r[vi].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k[:60]}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot * 100:.1f}% |")


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = [h.index(w) for w in WANT if w in h]
    print("| kernel | " + " | ".join(f"{h[i]} ({units[i]})" for i in idx) + " |")
    print("|---" * (len(idx) + 1) + "|")
    for r in rows[2:]:
        print(f"| `{r[h.index('Kernel Name')][:40]}` | " + " | ".join(r[i] for i in idx) + " |")


if __name__ == "__main__":
    print("## launch list (ncu --metrics gpu__time_duration.sum; cold-cache, serialised: compare shares)\n")
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        print("\n## ncu --set full (per launch)\n")
        full(sys.argv[2])
