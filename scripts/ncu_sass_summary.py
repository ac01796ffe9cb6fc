"""Summarise an ncu --page source --print-source sass CSV: hottest
instructions by stall samples and by executed count, and per-opcode totals.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    python scripts/ncu_sass_summary.py sass.csv [--top 40]
"""

from __future__ import annotations

import argparse
import collections
import csv


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    with open(args.csv) as f:
        rows = list(csv.reader(f))
    hdr = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]

    def num(r, name):
        try:
            return float(r[col[name]] or 0)
        except (KeyError, ValueError):
            return 0.0

    total_s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body)
    total_i = sum(num(r, "Instructions Executed") for r in body)
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.Counter()
    for r in body:
        for h in stall_cols:
            agg[h] += num(r, h)
    print(f"instructions executed (warp-level): {total_i:.3e}; stall samples: {total_s:.0f}")
    print("stall reasons:", ", ".join(f"{k[6:]} {v / max(total_s, 1):.1%}" for k, v in agg.most_common(10)))
    ops = collections.Counter()
    ops_s = collections.Counter()
    for r in body:
        op = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[col["Source"]].split()[1]
        ops[op] += num(r, "Instructions Executed")
        ops_s[op] += num(r, "Warp Stall Sampling (All Samples)")
    print("\nopcode            executed   share  stall-share")
    for op, n in ops.most_common(25):
        print(f"{op:16s} {n:10.3e}  {n / total_i:6.1%}  {ops_s[op] / max(total_s, 1):6.1%}")
    print(f"\ntop {args.top} instructions by stall samples:")
    hot = sorted(body, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[: args.top]
    for r in hot:
        reasons = sorted(((num(r, h), h[6:]) for h in stall_cols), reverse=True)[:2]
        print(f"{r[col['Address']]:>6} {num(r, 'Warp Stall Sampling (All Samples)') / max(total_s, 1):6.2%} "
              f"exec {num(r, 'Instructions Executed'):9.3e} {r[col['Source']][:60]:60s} "
              + " ".join(f"{n}:{v / max(total_s, 1):.1%}" for v, n in reasons))


if __name__ == "__main__":
    main()
