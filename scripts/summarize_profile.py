"""Write the committed profile summary for one ncu --set full capture.

    python scripts/summarize_profile.py gpurun_out/k2_TAG.ncu-rep profiles/rNN_k2_hotset.md \
        [--traffic-json profiles/k2_traffic.json] [--launches gpurun_out/launches.csv]

Reads the report with `ncu -i` (no GPU needed) and records: duration, DRAM
bytes (the `traffic` figure bench.py reports), L2 hit rate, issue/occupancy
numbers, the warp-stall breakdown and the per-opcode instruction mix.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
import sys


def ncu(rep: str, *args: str) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic-json")
    ap.add_argument("--launches")
    ap.add_argument("--workload", default="C2 workload")
    args = ap.parse_args()

    raw = ncu(args.rep, "--page", "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = {h: (v, u) for h, v, u in zip(hdr, vals, units)}

    def val(k, scale=1.0):
        v, u = m[k]
        x = float(v.replace(",", ""))
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}
        return x * mult.get(u, 1.0) * scale

    dur = val("gpu__time_duration.sum")
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    lines = [f"# ncu summary: {m['Kernel Name'][0] if 'Kernel Name' in m else 'kernel'}", "",
             f"source report: `{args.rep}` (ncu --set full --clock-control none, 1 launch, {args.workload})", "",
             "| metric | value |", "|---|---|"]
    rows = [
        ("duration (ms, serialised, cold-ish)", f"{dur * 1e3:.3f}"),
        ("dram__bytes_read.sum (GB)", f"{rd / 1e9:.3f}"),
        ("dram__bytes_write.sum (MB)", f"{wr / 1e6:.2f}"),
        ("DRAM GB/s (traffic / duration)", f"{(rd + wr) / dur / 1e9:.0f}"),
    ]
    for k, label in [("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
                     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
                     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
                     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of max"),
                     ("launch__registers_per_thread", "registers/thread"),
                     ("smsp__inst_executed.sum", "warp instructions executed"),
                     ("launch__grid_size", "grid"), ("launch__block_size", "block")]:
        if k in m:
            rows.append((label, m[k][0]))
    lines += [f"| {a} | {b} |" for a, b in rows]

    sass = ncu(args.rep, "--page", "source", "--print-source", "sass")
    shdr = sass[1]
    col = {h: i for i, h in enumerate(shdr)}
    body = [r for r in sass[2:] if len(r) == len(shdr)]

    def num(r, name):
        try:
            return float(r[col[name]] or 0)
        except (KeyError, ValueError):
            return 0.0

    stall_cols = [h for h in shdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body) or 1.0
    agg = collections.Counter()
    ops = collections.Counter()
    for r in body:
        for h in stall_cols:
            agg[h[6:]] += num(r, h)
        toks = r[col["Source"]].split()
        if toks:
            ops[toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]] += num(r, "Instructions Executed")
    lines += ["", "## Warp-stall breakdown (sampled)", "", "| reason | share |", "|---|---|"]
    lines += [f"| {k} | {v / tot:.1%} |" for k, v in agg.most_common(10)]
    itot = sum(ops.values()) or 1.0
    lines += ["", "## Instruction mix (warp-level executed)", "", "| opcode | executed | share |", "|---|---|---|"]
    lines += [f"| {k} | {v:.3e} | {v / itot:.1%} |" for k, v in ops.most_common(15)]

    if args.launches:
        with open(args.launches) as f:
            text = f.read()
        start = text.find('"ID"')
        lrows = list(csv.reader(io.StringIO(text[start:])))
        lh = lrows[0]
        c = {h: i for i, h in enumerate(lh)}
        per = collections.defaultdict(list)
        for r in lrows[1:]:
            if len(r) == len(lh) and r[c["Metric Name"]] == "gpu__time_duration.sum":
                name = r[c["Kernel Name"]].split("(")[0]
                v = float(r[c["Metric Value"]].replace(",", ""))
                unit = r[c["Metric Unit"]]
                per[name].append(v * {"ms": 1e3, "us": 1.0, "ns": 1e-3}.get(unit, 1.0))
        lines += ["", "## Launch list (gpu__time_duration.sum, cold, serialised)", "",
                  "| kernel | launches | mean us | total us |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} |")

    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if args.traffic_json:
        with open(args.traffic_json, "w") as f:
            name = m["Kernel Name"][0] if "Kernel Name" in m else ""
            kernel = next((k for k in ("k2_relay", "k2_hotset", "k2_pair", "k2_dense") if k in name), name)
            l2_sectors = val("lts__t_sectors_srcunit_tex_op_read.sum") if "lts__t_sectors_srcunit_tex_op_read.sum" in m else None
            json.dump({"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                       "l2_read_sectors_per_launch": l2_sectors,
                       "duration_s": dur, "report": args.rep, "kernel": kernel}, f, indent=1)
    print("\n".join(lines[:14]))


if __name__ == "__main__":
    sys.exit(main())
