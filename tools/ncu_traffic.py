"""Per-kernel time and DRAM bytes of the last search in an ncu CSV launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --cache-control none --clock-control none --csv \
        python tools/probes/one_search.py c2 1 800 > launches.csv
    python tools/ncu_traffic.py launches.csv c2 [--out profiles/c2_rerank_traffic.json]

The last search = the launches from the last ``k_slice_rows`` (a search's first kernel;
the index build's own slicing comes earlier) to the end.  Prints the launch table and
writes the re-rank stage's bytes / time (the bench's ``roofline.traffic`` source).
"""

from __future__ import annotations

import argparse
import csv
import json
from collections import OrderedDict

RERANK = ("k_rr_items", "k_rr_groups", "k_rr_screen", "k_rr_thresh", "k_interleave_queries",
          "k_rerank_sparse", "k_rerank_cluster", "k_topk_final")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("workload")
    ap.add_argument("--out")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 12 and r[0].isdigit()]
    launches = OrderedDict()
    for r in rows:
        key = (int(r[0]), r[4])
        launches.setdefault(key, {})[r[-3]] = float(r[-1].replace(",", ""))
    items = [(k[1], v) for k, v in launches.items()]
    start = max(i for i, (n, _) in enumerate(items) if n.startswith("k_slice_rows"))
    search = items[start:]
    tot_us = 0.0
    per = OrderedDict()
    print(f"{'us':>9} {'MB':>9}  kernel")
    for name, m in search:
        us = m.get("gpu__time_duration.sum", 0.0) / 1e3
        mb = (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6
        tot_us += us
        short = name.split("(")[0].replace("void ", "").split("<")[0]
        print(f"{us:9.1f} {mb:9.1f}  {name[:90]}")
        if short.startswith(RERANK):
            p = per.setdefault(short, {"bytes": 0.0, "us": 0.0})
            p["bytes"] += mb * 1e6
            p["us"] += us
    print(f"{tot_us:9.1f}            serialised total")
    out = {
        "kernel": " + ".join(per) + " (the re-rank stage)",
        "bytes_per_launch": int(sum(p["bytes"] for p in per.values())),
        "per_kernel": per,
        "serialised_us": round(sum(p["us"] for p in per.values()), 1),
        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  f"--cache-control none --clock-control none, one {a.workload.upper()} search ({a.csv})",
    }
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
        print("wrote", a.out)


if __name__ == "__main__":
    main()
