"""Top SASS lines by a stall reason:  python scripts/ncu_stalls.py REP [reason=stall_long_sb] [N]"""
import csv, subprocess, sys
rep = sys.argv[1]; reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"; n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines())); h = rows[1]; data = rows[2:]; ix = {k: i for i, k in enumerate(h)}
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
tot = sum(f(r, reason) for r in data); allst = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"{reason}: {tot:.0f} samples of {allst:.0f} ({100*tot/max(allst,1):.1f}%)")
for i, r in sorted(enumerate(data), key=lambda x: -f(x[1], reason))[:n]:
    print("%6d %7.0f %5.1f%%  %s" % (i, f(r, reason), 100 * f(r, reason) / max(tot, 1), r[ix["Source"]][:80]))
