"""Summarise an ncu report: per kernel duration, DRAM bytes/throughput, issue, occupancy, top stalls.

    python tools/ncu_brief.py gpurun_out/x.ncu-rep
"""
import csv
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        st = {}
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        top = sorted(((v, k) for k, v in st.items()), reverse=True)[:6]
        name = d.get("Kernel Name", "?")[:60]
        u = lambda k: units.get(k, "")  # noqa: E731
        print(f"{name}\n  dur {d.get('gpu__time_duration.sum')} {u('gpu__time_duration.sum')}"
              f"  dram rd {d.get('dram__bytes_read.sum')} {u('dram__bytes_read.sum')}"
              f" wr {d.get('dram__bytes_write.sum')} {u('dram__bytes_write.sum')}"
              f"  dram% {d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}"
              f"  issue% {d.get('sm__inst_issued.avg.pct_of_peak_sustained_active')}"
              f"  occ% {d.get('sm__warps_active.avg.pct_of_peak_sustained_active')}")
        print("  stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for v, k in top))


if __name__ == "__main__":
    main(sys.argv[1])
