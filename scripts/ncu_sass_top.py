"""Hottest SASS instructions of an `ncu --page source --csv --print-source
cuda,sass` export, in address order around the top stall sites.

    python scripts/ncu_sass_top.py src.csv [--top 40]
"""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=40)
args = ap.parse_args()
rows = []
hdr = None
with open(args.csv, errors="replace") as f:
    for r in csv.reader(f):
        if r and r[0] == "Line No":
            hdr = r
            col = {h: i for i, h in enumerate(hdr)}
            stall_cols = [(h, i) for h, i in col.items() if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or len(r) != len(hdr) or r[0]:
            continue  # sass rows have an empty line number
        try:
            addr = int(r[2], 16)
            ss = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
            ie = float(r[col["Instructions Executed"]] or 0)
        except ValueError:
            continue
        reasons = sorted(((float(r[i] or 0), h[6:]) for h, i in stall_cols), reverse=True)[:2]
        rows.append((addr, r[3].strip(), ss, ie, reasons))
tot = sum(x[2] for x in rows) or 1
for addr, sass, ss, ie, rs in sorted(rows, key=lambda x: -x[2])[: args.top]:
    why = ", ".join(f"{n} {c / max(ss, 1):.0%}" for c, n in rs if c)
    print(f"{addr & 0xFFFF:05x} {ss / tot:6.1%} {ie / 1e6:7.1f}M  {sass[:60]:60s} [{why}]")
