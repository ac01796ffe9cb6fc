"""Measurements for the non-headline BASELINE.json configs on one B200.

    python scripts/sweep.py [--quick] [--out profiles/r01_sweep.json]

  C3  1M trials x 1000 events, 16-layer portfolio (seed 2066, 32-ELT pool,
      15 ELTs per layer; even layers Per-Occurrence XL, odd layers Aggregate
      XL, terms from the generator), layers run back to back, then the
      on-device portfolio roll-up and K3 on it.
  C4  10M trials x 1000 events x 15 ELTs (40 GB of ids generated on the
      device -- uniform ids, like the reference generator), hot-set kernel
      and the dense uncompacted kernel.
  C5  events/trial E in {100..5000} x ELTs J in {1..64}, T = 1e9 / E trials,
      catalog 2M: trials/s, K2 ms, algorithmic and compulsory GB/s.

Times are CUDA-event times of the K2 launches (inputs resident in HBM),
median of 5 after 2 warm-ups.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1308_2066_b200 import _native  # noqa: E402
from paper_1308_2066_b200.direct_access import TableSet  # noqa: E402
from paper_1308_2066_b200.portfolio import Layer, LayerTerms  # noqa: E402
from paper_1308_2066_b200.resident import DeviceYearEventTable  # noqa: E402
from paper_1308_2066_b200.risk import order_stats, rollup_device  # noqa: E402
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_layer  # noqa: E402

CATALOG = 2_000_000
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def device_yet(trials: int, events: int, seed: int) -> DeviceYearEventTable:
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    ids = torch.randint(1, CATALOG + 1, (trials * events + 4,), dtype=torch.int32, device="cuda", generator=g)
    offsets = np.arange(trials + 1, dtype=np.int64) * events
    d_off = torch.from_numpy(offsets).cuda()
    return DeviceYearEventTable.from_device(CATALOG, ids[: trials * events], d_off, offsets)


def time_k2(dyet, plan, terms, reps: int = 5, warm: int = 2, variant: str = "auto") -> float:
    out = torch.empty(dyet.trial_count, dtype=torch.float64, device="cuda")
    for _ in range(warm):
        dyet.simulate_device(plan, terms, out=out, variant=variant)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dyet.simulate_device(plan, terms, out=out, check=False, variant=variant)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def c5(quick: bool) -> list[dict]:
    spec = GeneratorSpec(seed=2066, catalog_size=CATALOG, elt_count=64, elt_size_range=(10_000, 30_000))
    pool = [generate_elt(spec, i) for i in range(64)]
    terms = LayerTerms(500.0, 10_000.0, 140_000.0, 66_000.0)
    es = [100, 1000, 5000] if quick else [100, 250, 500, 1000, 2000, 5000]
    js = [1, 15, 64] if quick else [1, 2, 4, 8, 15, 16, 32, 64]
    rows = []
    for e in es:
        t = int(1e9 // e)
        dyet = device_yet(t, e, seed=e)
        for j in js:
            tset = TableSet.from_elts(pool[:j], CATALOG)
            plan = tset.plan(*tset.selection_arrays(None))
            info = _native.plan_info(plan)
            ms = time_k2(dyet, plan, terms)
            alg = t * (12 + 4 * e * (1 + j))
            comp = t * (4 * e + 16)
            rows.append({"events": e, "elts": j, "trials": t, "k2_ms": ms, "trials_per_s": t / (ms / 1e3),
                         "hot_events": info.hot_events, "entries": info.entries,
                         "algorithmic_gbs": alg / (ms / 1e3) / 1e9, "algorithmic_frac": alg / (ms / 1e3) / 1e9 / PEAK,
                         "compulsory_gbs": comp / (ms / 1e3) / 1e9, "compulsory_frac": comp / (ms / 1e3) / 1e9 / PEAK})
            print(json.dumps(rows[-1]), flush=True)
            del tset, plan
        del dyet
        torch.cuda.empty_cache()
    return rows


def c4(quick: bool) -> dict:
    trials = 2_000_000 if quick else 10_000_000
    spec = GeneratorSpec(seed=2066, catalog_size=CATALOG, elt_count=15, elt_size_range=(10_000, 30_000))
    elts = [generate_elt(spec, i) for i in range(15)]
    tset = TableSet.from_elts(elts, CATALOG)
    plan = tset.plan(*tset.selection_arrays(None))
    dyet = device_yet(trials, 1000, seed=44)
    terms = LayerTerms(500.0, 10_000.0, 140_000.0, 66_000.0)
    ms = time_k2(dyet, plan, terms, reps=3)
    # also the dense, uncompacted layout (every lookup a
    # float64 gather from the 240 MB tables: the exceeds-L2 regime)
    dms = time_k2(dyet, plan, terms, reps=1, warm=1, variant="dense")
    alg = trials * (12 + 4 * 1000 * 16)
    out = {"trials": trials, "events": 1000, "elts": 15, "k2_ms": ms, "trials_per_s": trials / (ms / 1e3),
           "id_bytes": trials * 4000, "compulsory_frac": trials * 4016 / (ms / 1e3) / 1e9 / PEAK,
           "algorithmic_frac": alg / (ms / 1e3) / 1e9 / PEAK,
           "dense": {"k2_ms": dms, "trials_per_s": trials / (dms / 1e3),
                     "algorithmic_frac": alg / (dms / 1e3) / 1e9 / PEAK,
                     "note": "k2_dense: the literal reference loop over dense float64 rows"}}
    print(json.dumps(out), flush=True)
    del dyet
    torch.cuda.empty_cache()
    return out


def c3(quick: bool) -> dict:
    trials = 200_000 if quick else 1_000_000
    spec = GeneratorSpec(seed=2066, catalog_size=CATALOG, elt_count=32, elt_size_range=(10_000, 30_000),
                         layer_count=16, elts_per_layer=15)
    pool = [generate_elt(spec, i) for i in range(32)]
    layers = []
    for i in range(16):
        g = generate_layer(spec, i, pool)
        t = g.terms
        terms = LayerTerms(t.occ_retention, t.occ_limit, 0.0, math.inf) if i % 2 == 0 else \
            LayerTerms(0.0, math.inf, t.agg_retention, t.agg_limit)
        layers.append(Layer(g.id, g.elts, terms))
    plans = []
    for lay in layers:
        ts = TableSet.from_elts(lay.elts, CATALOG)
        plans.append((ts, ts.plan(*ts.selection_arrays(None))))
    dyet = device_yet(trials, 1000, seed=33)
    outs = [torch.empty(trials, dtype=torch.float64, device="cuda") for _ in layers]

    def step():
        for (ts, plan), lay, o in zip(plans, layers, outs):
            dyet.simulate_device(plan, lay.terms, out=o, check=False)
        total = rollup_device(outs)
        return order_stats(total, [10.0, 50.0, 100.0, 250.0])

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    reps = 3
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        res = step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    # fused: one pass over the YET for all 16 layers
    from paper_1308_2066_b200.engine import layer_pool, simulate_layers_device

    pool_elts, masks = layer_pool(layers)
    ptset = TableSet.from_elts(pool_elts, CATALOG)
    fused = torch.empty((16, trials), dtype=torch.float64, device="cuda")

    def fused_step():
        simulate_layers_device(dyet, ptset, masks, [l.terms for l in layers], out=fused)
        total = rollup_device([fused[i] for i in range(16)])
        return order_stats(total, [10.0, 50.0, 100.0, 250.0])

    for _ in range(2):
        fres = fused_step()
    same = all(torch.equal(fused[i], outs[i]) for i in range(16))
    a.record()
    for _ in range(reps):
        fres = fused_step()
    b.record()
    torch.cuda.synchronize()
    fms = a.elapsed_time(b) / reps

    def pre_step():  # per-event occurrence table (SURVEY 8(f) rows 2 + 4)
        simulate_layers_device(dyet, ptset, masks, [l.terms for l in layers], out=fused, precombine=True)
        total = rollup_device([fused[i] for i in range(16)])
        return order_stats(total, [10.0, 50.0, 100.0, 250.0])

    for _ in range(2):
        pre_step()
    pre_same = all(torch.equal(fused[i], outs[i]) for i in range(16))
    a.record()
    for _ in range(reps):
        pre_step()
    b.record()
    torch.cuda.synchronize()
    pms = a.elapsed_time(b) / reps
    out = {"trials": trials, "layers": 16, "step_ms": ms, "trials_per_s": trials / (ms / 1e3),
           "layer_trials_per_s": 16 * trials / (ms / 1e3), "portfolio_pml": list(map(float, res[0])),
           "note": "16 K2 launches (one per layer) + k3_rollup + K3 per step; unfused",
           "fused_step_ms": fms, "fused_trials_per_s": trials / (fms / 1e3),
           "fused_layer_trials_per_s": 16 * trials / (fms / 1e3), "fused_bitwise_equal_unfused": bool(same),
           "fused_portfolio_pml": list(map(float, fres[0])),
           "precombined_step_ms": pms, "precombined_layer_trials_per_s": 16 * trials / (pms / 1e3),
           "precombined_bitwise_equal_unfused": bool(pre_same)}
    print(json.dumps(out), flush=True)
    return out


def validate(quick: bool) -> dict:
    """validate_portfolio's YET checks on the device (K0,
    timestamps streamed from the host) vs the host numpy path."""
    from paper_1308_2066_b200.portfolio import YearEventTable, validate_portfolio
    from paper_1308_2066_b200.synth import bulk_yet

    trials = 100_000 if quick else 1_000_000
    yet = bulk_yet(7, CATALOG, 0, trials, 1000, threads=os.cpu_count() or 8)
    ts = np.tile(np.linspace(0.0, 1.0, 1000), trials)
    full = YearEventTable(CATALOG, yet.event_ids, ts, yet.offsets)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dyet = DeviceYearEventTable(full)
    viol = dyet.yet_violations()
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    sample = full.head(100_000)
    t0 = time.perf_counter()
    host_viol = validate_portfolio([], sample)
    host_s = (time.perf_counter() - t0) * trials / 100_000
    out = {"trials": trials, "events": 1000, "device_seconds_incl_h2d_of_ids_and_timestamps": dev_s,
           "host_numpy_seconds_extrapolated_from_100k": host_s, "violations": [str(v) for v in viol],
           "host_violations_on_sample": [str(v) for v in host_viol]}
    print(json.dumps(out), flush=True)
    return out


# The reference's own linear-scaling sweeps (pkg/src/aggrisk/bench.py:159-230,
# base spec :177-184; asserted by tests/test_acceptance.py:121-137) with the
# seconds its recorded run reports for its compiled CPU engine, one worker
# (pkg/test_output.txt:244-253).
REF_RECORDED = {
    "trials": {20_000: 0.225, 40_000: 0.466, 60_000: 0.712, 80_000: 0.963, 100_000: 1.201},
    "events_per_trial": {800: 1.132, 900: 1.249, 1000: 1.457, 1100: 1.547, 1200: 1.774},
    "elts_per_layer": {3: 0.118, 6: 0.240, 9: 0.382, 12: 0.518, 15: 0.685},
    "layers": {1: 0.114, 2: 0.228, 3: 0.346, 4: 0.441, 5: 0.573},
}


def refsweeps(quick: bool) -> dict:
    """The same four sweeps through the same API (run_aggregate_analysis_with_
    stats, RunStats.sim_seconds, min over 3 interleaved rounds), inputs from
    the reference generator restatement (byte-identical YET/ELTs)."""
    from paper_1308_2066_b200.engine import run_aggregate_analysis_with_stats
    from paper_1308_2066_b200.synth import generate_yet

    base = dict(seed=7, catalog_size=50_000, trial_count=20_000, events_per_trial_range=(1000, 1000),
                elt_count=15, elt_size_range=(10_000, 30_000))

    def flat(elts, lid="bench"):
        return Layer(lid, tuple(elts), LayerTerms())

    plans = {}
    spec = GeneratorSpec(**{**base, "trial_count": 100_000, "elt_count": 6})
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(6)]
    plans["trials"] = [(v, [flat(elts)], yet.head(v)) for v in REF_RECORDED["trials"]]
    spec = GeneratorSpec(**{**base, "events_per_trial_range": (1200, 1200), "trial_count": 40_000})
    full = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(15)]
    ev = full.event_ids.reshape(-1, 1200)
    ts = full.timestamps.reshape(-1, 1200)
    from paper_1308_2066_b200.portfolio import YearEventTable

    plans["events_per_trial"] = [
        (v, [flat(elts)], YearEventTable(full.catalog_size, np.ascontiguousarray(ev[:, :v]).ravel(),
                                         np.ascontiguousarray(ts[:, :v]).ravel(),
                                         np.arange(ev.shape[0] + 1, dtype=np.int64) * v))
        for v in REF_RECORDED["events_per_trial"]]
    spec = GeneratorSpec(**base)
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(15)]
    plans["elts_per_layer"] = [(v, [flat(elts[:v])], yet) for v in REF_RECORDED["elts_per_layer"]]
    spec = GeneratorSpec(**{**base, "elt_count": 3})
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(3)]
    plans["layers"] = [(v, [flat(elts, f"bench-{i}") for i in range(v)], yet) for v in REF_RECORDED["layers"]]

    out = {}
    for name, plan in plans.items():
        best = {}
        for _ in range(3):  # interleaved rounds, minimum per point (reference bench.py:113-140)
            for v, layers, y in plan:
                _, st = run_aggregate_analysis_with_stats(layers, y)
                best[v] = min(best.get(v, math.inf), st.sim_seconds)
        xs = np.array(sorted(best), dtype=np.float64)
        ys = np.array([best[v] for v in sorted(best)])
        fit = np.polyfit(xs, ys, 1)
        r2 = 1.0 - float(np.sum((ys - np.polyval(fit, xs)) ** 2) / np.sum((ys - ys.mean()) ** 2))
        out[name] = {"points": [{"value": int(v), "sim_seconds": best[v],
                                 "reference_recorded_seconds": REF_RECORDED[name][v],
                                 "speedup": REF_RECORDED[name][v] / best[v]} for v in sorted(best)],
                     "r2": r2}
        print(json.dumps({name: out[name]}), flush=True)
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--only", default="c3,c4,c5")
    args = ap.parse_args()
    res = {"device": torch.cuda.get_device_name(), "peak_hbm_gbs": PEAK, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ")}
    for name in args.only.split(","):
        res[name] = globals()[name](args.quick)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
