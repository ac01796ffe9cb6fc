"""SASS basic-block view of an ncu source export: consecutive instructions
with the same execution count are merged into blocks, so per-chunk /
per-batch / per-trial costs (instructions x executions) stand out.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    python scripts/ncu_blocks.py sass.csv [min_instructions] [lo_hex hi_hex]

With an address range (offsets from the kernel start, hex) the instructions
of that range are listed with their counts and stall samples.
"""
import csv
import sys


def main() -> None:
    rows = []
    with open(sys.argv[1]) as f:
        r = csv.reader(f)
        next(r)
        hdr = next(r)
        ia = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        for x in r:
            if len(x) < ia:
                continue
            rows.append((int(x[0], 16), x[1].strip(), float(x[ia] or 0), float(x[ss] or 0)))
    base = rows[0][0]
    tot = sum(r[2] for r in rows)
    tst = sum(r[3] for r in rows) or 1.0
    print("total %.4g warp instructions, %d stall samples" % (tot, tst))
    blocks, cur = [], None
    for a, s, n, st in rows:
        if cur and abs(cur[2] - n) < 1:
            cur[1] = a
            cur[3] += 1
            cur[4] += st
        else:
            if cur:
                blocks.append(cur)
            cur = [a, a, n, 1, st]
    blocks.append(cur)
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e7
    for b in blocks:
        if b[2] * b[3] > thr:
            print(f"{b[0] - base:5x}-{b[1] - base:5x} n={b[2] / 1e6:7.2f}M x{b[3]:3d} = {b[2] * b[3] / 1e6:8.1f}M "
                  f"({100 * b[2] * b[3] / tot:4.1f}%) stall {100 * b[4] / tst:4.1f}%")
    if len(sys.argv) > 4:
        lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
        for a, s, n, st in rows:
            if lo <= a - base <= hi:
                print(f"{a - base:5x} {n / 1e6:6.2f}M {st:6.0f} {s}")


if __name__ == "__main__":
    main()
