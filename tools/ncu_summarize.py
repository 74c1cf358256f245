"""Summarise an ncu --set full report of BC kernel (bc_team_kernel / bc_sources_kernel) into markdown.

    python tools/ncu_summarize.py gpurun_out/prof.ncu-rep --sources 296 > profiles/rNN_x.md
"""
import argparse
import collections
import csv
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
           "lts__t_sectors_srcunit_tex_op_read.sum", "dram__sectors_read.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def lines(rep, top):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[2]
    ist, il2 = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("L2 Theoretical Sectors Global")
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    for r in rows[3:]:
        if len(r) <= ist:
            continue
        a = agg[r[0]]
        for i, j in ((0, ist), (1, il2)):
            try:
                a[i] += float(r[j])
            except ValueError:
                pass
        a[2] = r[1]
    ts = sum(a[0] for a in agg.values()) or 1
    tl = sum(a[1] for a in agg.values()) or 1
    return [(k, 100 * a[0] / ts, 100 * a[1] / tl, a[2].strip()) for k, a in
            sorted(agg.items(), key=lambda x: -x[1][0])[:top]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--sources", type=int, required=True, help="sources processed by the profiled launch")
    ap.add_argument("--top", type=int, default=15)
    a = ap.parse_args()
    m = raw(a.rep)
    print(f"### `{a.rep.split('/')[-1]}` ({a.sources} sources in the profiled launch)\n")
    print("| metric | value | unit |\n|---|---|---|")
    for k in METRICS:
        if k in m:
            print(f"| {k} | {m[k][0]} | {m[k][1]} |")
    rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
    wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
    scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    tot = rd * scale[m["dram__bytes_read.sum"][1]] + wr * scale[m["dram__bytes_write.sum"][1]]
    print(f"\nDRAM traffic per source: **{tot / a.sources / 1e9:.4g} GB** (read+write)\n")
    print("Top source lines by warp-stall samples (line '' = inline PTX loads without line info):\n")
    print("| line | stall % | L2 sectors % | source |\n|---|---|---|---|")
    for k, s, l2, src in lines(a.rep, a.top):
        print(f"| {k} | {s:.1f} | {l2:.1f} | `{src[:80]}` |")


if __name__ == "__main__":
    main()
