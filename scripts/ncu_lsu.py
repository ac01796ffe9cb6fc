"""Per-SM LSU wavefront / instruction accounting of one ncu report (source page, SASS):
    python scripts/ncu_lsu.py REPORT.ncu-rep [--top N]"""
import csv, collections, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
for r in data:
    s = r[ix["Source"]].strip()
    parts = s.split()
    if not parts: continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    a = agg[op]
    a[0] += f(r, "L1 Wavefronts Shared") / 148; a[1] += f(r, "L1 Tag Requests Global") / 148
    a[2] += f(r, "Instructions Executed") / 148; a[3] += 1
tot = [sum(a[i] for a in agg.values()) for i in range(3)]
print("per SM: shared wavefronts %.0f  global tag requests %.0f  LSU total %.0f  warp instructions %.0f"
      % (tot[0], tot[1], tot[0] + tot[1], tot[2]))
for op, (ws, tg, ie, n) in sorted(agg.items(), key=lambda x: -(x[1][0] + x[1][1]))[:12]:
    print("  %-26s wavefronts %9.0f  tag %9.0f  inst %9.0f  sites %d" % (op, ws, tg, ie, n))
if top:
    items = sorted(data, key=lambda r: -(f(r, "L1 Wavefronts Shared") + f(r, "L1 Tag Requests Global")))[:top]
    for r in items:
        print("%9.0f %9.0f %9.0f  %s" % (f(r, "L1 Wavefronts Shared") / 148, f(r, "L1 Tag Requests Global") / 148,
                                       f(r, "Instructions Executed") / 148, r[ix["Source"]][:70]))
