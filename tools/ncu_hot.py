"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).

    python tools/ncu_hot.py report.ncu-rep kernel_regex [n]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    recs = []
    fname = ""
    for r in rows:
        if r and r[0] in ("File Name", "File Path"):
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[2] == "-":
            recs.append((fname, r))
    if not hdr:
        print(out[:2000])
        return
    si = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[si] or 0) for _, r in recs) or 1.0
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for f, r in sorted(recs, key=lambda x: -float(x[1][si] or 0))[:n]:
        stalls = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        st = " ".join(f"{name}:{v / tot * 100:.0f}%" for v, name in stalls if v > 0)
        print(f"{float(r[si]) / tot * 100:5.1f}% {f}:{r[0]:>4} {r[1].strip()[:70]:70s} {st}")


if __name__ == "__main__":
    main()
