"""Per-source-line view of an ncu report: instructions executed and stall
samples (with the dominant stall reasons), across all files of the kernel.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [--top 25] [--by inst|stall]
"""
import argparse
import collections
import csv
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--by", default="stall")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr = "?", None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1]
    for i, h in enumerate(hdr):
        if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or (h.startswith("stall_") and "Not Issued" not in h):
            try:
                agg[key][h] += float(r[i])
            except ValueError:
                pass
tot_s = sum(c["Warp Stall Sampling (All Samples)"] for c in agg.values()) or 1
tot_i = sum(c["Instructions Executed"] for c in agg.values()) or 1
k = "Warp Stall Sampling (All Samples)" if a.by == "stall" else "Instructions Executed"
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.4g}")
for key, c in sorted(agg.items(), key=lambda x: -x[1][k])[: a.top]:
    reasons = sorted(((v, h[6:]) for h, v in c.items() if h.startswith("stall_") and v), reverse=True)[:3]
    rs = " ".join(f"{n}:{100 * v / max(1, c['Warp Stall Sampling (All Samples)']):.0f}%" for v, n in reasons)
    print(f"{key[0][:14]:14s}:{key[1]:4d} stall {100 * c['Warp Stall Sampling (All Samples)'] / tot_s:5.1f}% "
          f"inst {100 * c['Instructions Executed'] / tot_i:5.1f}% [{rs}] {src[key].strip()[:70]}")
