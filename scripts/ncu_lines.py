"""Per-source-line summary of an `ncu --page source --csv --print-source
cuda,sass` export: executed instructions, stall-sample share and top stall
reasons, hottest lines first.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_lines.py src.csv [--top 30] [--by instr|stall]
"""

from __future__ import annotations

import argparse
import collections
import csv


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--by", choices=("instr", "stall"), default="stall")
    args = ap.parse_args()
    cur = None
    hdr = None
    col: dict[str, int] = {}
    agg = collections.defaultdict(lambda: [0.0, 0.0, "", collections.Counter()])
    tot_i = tot_s = 0.0
    with open(args.csv) as f:
        for r in csv.reader(f):
            if len(r) == 2 and r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r and r[0] == "Line No":
                hdr = r
                col = {h: i for i, h in enumerate(hdr)}
                continue
            if hdr is None or len(r) != len(hdr) or not r[0]:
                continue
            try:
                ie = float(r[col["Instructions Executed"]] or 0)
                ss = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
            except (KeyError, ValueError):
                continue
            a = agg[(cur, int(r[0]))]
            a[0] += ie
            a[1] += ss
            a[2] = r[1].strip()[:80]
            for h, i in col.items():
                if h.startswith("stall_") and "Not Issued" not in h:
                    try:
                        a[3][h[6:]] += float(r[i] or 0)
                    except ValueError:
                        pass
            tot_i += ie
            tot_s += ss
    print(f"instructions {tot_i:.3e}  stall samples {tot_s:.0f}")
    key = 0 if args.by == "instr" else 1
    for (fname, line), v in sorted(agg.items(), key=lambda kv: -kv[1][key])[: args.top]:
        top = ", ".join(f"{k} {c / max(v[1], 1):.0%}" for k, c in v[3].most_common(2))
        print(f"{fname[:16]:16s}{line:5d} {v[0] / 1e6:8.1f}M  stall {v[1] / max(tot_s, 1):6.1%}  [{top}]  {v[2]}")


if __name__ == "__main__":
    main()
