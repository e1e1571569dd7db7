"""Summarise ncu outputs brought back in gpurun_out/ into a markdown file under profiles/.

usage: python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <out.md> [title]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg, unit = {}, ""
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
        unit = r[ui]
    tot = sum(sum(v) for v in agg.values())
    out = [f"| kernel | launches | mean ({unit}) | total ({unit}) | share |", "|---|---|---|---|---|"]
    for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{n}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |")
    return "\n".join(out)


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0]
        out.append(f"\n**{name}** (grid {row[h.index('launch__grid_size')] if 'launch__grid_size' in h else '?'})\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"| {m} | {row[i]} | {units[i]} |")
    return "\n".join(out)


if __name__ == "__main__":
    lc, rep, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else "ncu summary"
    body = [f"# {title}\n", "## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)\n",
            "Cold-cache, serialised: compare shares, not absolutes.\n", launches(lc),
            "\n## `ncu --set full` of the top kernel\n", full(rep)]
    open(dst, "w").write("\n".join(body) + "\n")
    print(open(dst).read())
