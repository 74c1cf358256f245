"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/ncu_launches.py gpurun_out/launches.csv
"""
import csv
import sys

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0}
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = {}
for r in rows[start + 1:]:
    if len(r) > vi:
        k = r[ki].split("(")[0][:70]
        t = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        n, s = tot.get(k, (0, 0.0))
        tot[k] = (n + 1, s + t)
T = sum(s for _, s in tot.values())
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (n, s) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {s * 1e3:.2f} | {100 * s / T:.2f}% |")
