"""Where the entry point's sim_seconds go on a promoted (HBM-resident) YET:
plan build (K1), K2, YLT readback -- host wall clock around each, synchronised."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1308_2066_b200.engine import run_aggregate_analysis_with_stats
from paper_1308_2066_b200.portfolio import Layer, LayerTerms
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.resident import DeviceYearEventTable

spec = GeneratorSpec(seed=7, catalog_size=50_000, trial_count=100_000, events_per_trial_range=(1000, 1000),
                     elt_count=6, elt_size_range=(10_000, 30_000))
yet = generate_yet(spec)
elts = [generate_elt(spec, i) for i in range(15)]
dyet = DeviceYearEventTable(yet)
for J in (6, 12):
    layer = Layer("b", tuple(elts[:J]), LayerTerms())
    for r in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ts = TableSet.from_elts(layer.elts, 50_000)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        plan = ts.plan(*ts.selection_arrays(None))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        d = dyet.simulate_device(plan, layer.terms)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        h = d.cpu().numpy()
        t4 = time.perf_counter()
        _, st = run_aggregate_analysis_with_stats([layer], dyet)
        print(f"J={J}: tables {1e3*(t1-t0):.2f} plan {1e3*(t2-t1):.2f} k2 {1e3*(t3-t2):.2f} d2h {1e3*(t4-t3):.2f} ms"
              f" | entry sim {st.sim_seconds*1e3:.2f} build {st.build_seconds*1e3:.2f}", flush=True)

# a fresh promotion before every call, like run_aggregate_analysis on a host YET
layer = Layer("b", tuple(elts[:6]), LayerTerms())
ts = TableSet.from_elts(layer.elts, 50_000)
for r in range(4):
    t0 = time.perf_counter()
    dy = DeviceYearEventTable(yet)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan = ts.plan(*ts.selection_arrays(None))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    d = dy.simulate_device(plan, layer.terms)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    d2 = dy.simulate_device(plan, layer.terms)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    _, st = run_aggregate_analysis_with_stats([layer], yet)
    t5 = time.perf_counter()
    print(f"fresh: promote {1e3*(t1-t0):.1f} plan {1e3*(t2-t1):.2f} k2 {1e3*(t3-t2):.2f} k2 again {1e3*(t4-t3):.2f} ms"
          f" | entry(host yet) sim {st.sim_seconds*1e3:.2f} build {st.build_seconds*1e3:.2f} wall {1e3*(t5-t4):.0f}", flush=True)
    del dy
