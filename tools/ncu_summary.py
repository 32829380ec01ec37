"""Summarise ncu reports / launch lists into small committed text files under profiles/.

    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep > profiles/r01_x.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.txt
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("lts__t_sectors_srcunit_tex_lookup_hit.sum", "l2_hit_sectors"),
    ("lts__t_sectors_srcunit_tex_lookup_miss.sum", "l2_miss_sectors"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
]


def report(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    idx = {name: i for i, name in enumerate(hdr)}
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[idx["Kernel Name"]] if "Kernel Name" in idx else r[4]
        print(f"\n## {name[:100]}")
        for m, label in METRICS:
            if m in idx:
                print(f"  {label:16s} {r[idx[m]]:>18s} {units[idx[m]]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:6]
        print("  top stalls       " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top))


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(list)
    order = []
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        if name not in per:
            order.append(name)
        per[name].append(us)
    total = sum(sum(v) for v in per.values()) or 1.0
    print(f"# launch list ({path}); gpu__time_duration, cold-cache serialised (shares, not absolutes)")
    print(f"{'kernel':60s} {'n':>4s} {'mean_us':>10s} {'share':>7s}")
    for name in sorted(order, key=lambda n: -sum(per[n])):
        v = per[name]
        print(f"{name[:60]:60s} {len(v):4d} {sum(v) / len(v):10.1f} {100 * sum(v) / total:6.1f}%")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
