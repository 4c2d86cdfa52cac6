#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run HERE on the reports gpurun brought back).

  python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/r01_launches.md
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep        > profiles/r01_relax_full.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.max.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_red.sum", "lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_static",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def short(name: str) -> str:
    name = name.replace("void ", "").replace("hyt::", "")
    return name.split("(")[0]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit in ("msecond", "ms") else v
        rows.append((short(r["Kernel Name"]), us))
    tot = sum(u for _, u in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for n, u in rows:
        agg[n][0] += 1
        agg[n][1] += u
    print(f"# ncu launch list summary ({path})\n")
    print(f"{len(rows)} launches, {tot / 1e3:.2f} ms of serialized, cold-cache kernel time "
          "(ncu --metrics gpu__time_duration.sum --clock-control none; compare SHARES, not absolutes)\n")
    print("| kernel | launches | total ms | share | avg us |")
    print("|---|---:|---:|---:|---:|")
    for n, (c, u) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{n}` | {c} | {u / 1e3:.2f} | {u / tot * 100:.1f}% | {u / c:.1f} |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary ({path})\n")
    for r in rows[2:]:
        print(f"## `{short(r[hdr.index('Kernel Name')])}`\n")
        print("| metric | value | unit |")
        print("|---|---:|---|")
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {m} | {r[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
