"""Headline counters and the top warp-stall reasons of an ncu report.

    python scripts/ncu_headline.py rep.ncu-rep
"""
import csv
import subprocess
import sys


def main() -> None:
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, v = r[0], r[2]
    keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "lts__t_sector_hit_rate.pct"]
    for i, k in enumerate(h):
        if k in keys:
            print(k, v[i])
    st = [(float(v[i]), k) for i, k in enumerate(h)
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
          and v[i].replace(".", "", 1).isdigit()]
    tot = sum(x for x, _ in st) or 1.0
    for x, k in sorted(st, reverse=True)[:9]:
        print(f"  {k[33:]:30s} {100 * x / tot:5.1f}%")


if __name__ == "__main__":
    main()
