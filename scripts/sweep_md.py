"""Render a scripts/sweep.py JSON result as the committed markdown summary.

    python scripts/sweep_md.py gpurun_out/sweep_TAG.json profiles/rNN_sweep.md
"""
import json
import sys


def main() -> None:
    src, dst = sys.argv[1], sys.argv[2]
    d = json.load(open(src))
    peak = d["peak_hbm_gbs"]
    out = [f"# Sweeps (one B200, CUDA-event time of the K2 launch, median of 5) -- {d['when']}", "",
           f"device: {d['device']}; HBM peak used for fractions: {peak} GB/s (MEASURED_PEAKS.json)", ""]
    if "c3" in d:
        c = d["c3"]
        out += ["## C3 -- 1M trials x 1000 events, 16 layers (Per-Occurrence / Aggregate XL alternating) over a 32-ELT pool", "",
                f"- unfused (one K2 per layer) + roll-up + K3: {c['step_ms']:.2f} ms per step -> "
                f"{c['trials_per_s'] / 1e6:.1f} M portfolio-trials/s, {c['layer_trials_per_s'] / 1e6:.0f} M layer-trials/s",
                f"- fused (one pass over the ids for all 16 layers, `k2_layers`) + roll-up + K3: {c['fused_step_ms']:.2f} ms "
                f"-> {c['fused_trials_per_s'] / 1e6:.1f} M portfolio-trials/s, "
                f"{c['fused_layer_trials_per_s'] / 1e6:.0f} M layer-trials/s; every layer's YLT bitwise equal to the "
                f"unfused run: {c['fused_bitwise_equal_unfused']}",
                f"- portfolio PML at rp 10/50/100/250: {', '.join(f'{x:,.0f}' for x in c['fused_portfolio_pml'])}"]
        if "precombined_step_ms" in c:
            out += [f"- pre-combined fused pass (per-event table of the 16 occurrence values, K1-L; a separately "
                    f"reported work unit) + roll-up + K3: {c['precombined_step_ms']:.2f} ms -> "
                    f"{c['precombined_layer_trials_per_s'] / 1e6:.0f} M layer-trials/s; bitwise equal: "
                    f"{c['precombined_bitwise_equal_unfused']}"]
        out += [""]
    if "c4" in d:
        c = d["c4"]
        out += [f"## C4 -- {c['trials']:,} trials x {c['events']} events x {c['elts']} ELTs "
                f"({c['id_bytes'] / 1e9:.0f} GB of ids resident in HBM)", "",
                f"- K2 (hot set) {c['k2_ms']:.2f} ms -> {c['trials_per_s'] / 1e6:.0f} M trials/s "
                f"(compulsory-bytes roofline fraction {c['compulsory_frac']:.2f}; algorithmic {c['algorithmic_frac']:.2f})"]
        if "dense" in c:
            dd = c["dense"]
            out += [f"- dense uncompacted kernel (`k2_dense`: every occurrence reads all selected float64 losses, no "
                    f"hot set; 240 MB of tables, the SURVEY 8(d) \"exceeding L2\" regime, read through an event-major "
                    f"copy): {dd['k2_ms']:.0f} ms -> {dd['trials_per_s'] / 1e6:.1f} M "
                    f"trials/s (algorithmic fraction {dd['algorithmic_frac']:.2f}), "
                    f"{dd['k2_ms'] / c['k2_ms']:.0f}x slower than the hot-set kernel"]
        out += [""]
    if "c5" in d:
        out += ["## C5 -- events/trial E x ELTs J (T = 1e9/E trials, catalog 2M)", "",
                "| E | J | trials | K2 ms | M trials/s | hot events | algorithmic GB/s (frac) | compulsory GB/s (frac) |",
                "|---|---|---|---|---|---|---|---|"]
        for r in d["c5"]:
            out.append(f"| {r['events']} | {r['elts']} | {r['trials']:,} | {r['k2_ms']:.2f} | {r['trials_per_s'] / 1e6:.0f} "
                       f"| {r['hot_events']:,} | {r['algorithmic_gbs']:.0f} ({r['algorithmic_frac']:.2f}) "
                       f"| {r['compulsory_gbs']:.0f} ({r['compulsory_frac']:.2f}) |")
        out += [""]
    if "refsweeps" in d:
        out += ["## The reference's own linear-scaling sweeps (catalog 50k, 1000 events, identity terms)", "",
                "Same entry point and counter as the reference bench (`run_aggregate_analysis_with_stats`, "
                "`RunStats.sim_seconds`, min of 3 interleaved rounds); reference = its recorded run of the compiled "
                "CPU engine on one worker (`pkg/test_output.txt:244-253`).", "",
                "| sweep | point | reference s | this engine ms | speed-up |", "|---|---|---|---|---|"]
        for name, r in d["refsweeps"].items():
            for p in r["points"]:
                out.append(f"| {name} | {p['value']:,} | {p['reference_recorded_seconds']:.3f} | "
                           f"{p['sim_seconds'] * 1e3:.2f} | {p['speedup']:,.0f}x |")
            out.append(f"| {name} | R^2 of this engine's times | | {r['r2']:.4f} | |")
        out += [""]
    open(dst, "w").write("\n".join(out))


if __name__ == "__main__":
    main()
