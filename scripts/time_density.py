"""K2 variants vs table density: the reference's own bench shape (catalog
50k: nearly every event in several of the ELTs) up to the paper's (catalog
2M: 14% of events hot, ~1 table each).  ms per 100k trials x 1000 events.

    python scripts/time_density.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, bulk_yet
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.resident import DeviceYearEventTable
from paper_1308_2066_b200.portfolio import LayerTerms

T = 100_000
for cat, J in ((50_000, 15), (50_000, 6), (50_000, 3), (200_000, 15), (2_000_000, 15)):
    spec = GeneratorSpec(seed=7, catalog_size=cat, elt_count=J, elt_size_range=(10_000, 30_000))
    elts = [generate_elt(spec, i) for i in range(J)]
    dyet = DeviceYearEventTable(bulk_yet(7, cat, 0, T, 1000, threads=8))
    tset = TableSet.from_elts(elts, cat)
    sel = tset.selection_arrays(None)
    plan, pplan = tset.plan(*sel), tset.plan(*sel, precombine=True)
    info = _native.plan_info(plan)
    o = torch.empty(T, dtype=torch.float64, device="cuda")
    res = {}
    for name, p, var in (("hotset", plan, "hotset"), ("dense", plan, "dense"), ("precombined", pplan, "hotset")):
        for _ in range(2):
            dyet.simulate_device(p, LayerTerms(), out=o, variant=var, check=False)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(5):
            dyet.simulate_device(p, LayerTerms(), out=o, variant=var, check=False)
        ev[1].record()
        torch.cuda.synchronize()
        res[name] = round(ev[0].elapsed_time(ev[1]) / 5, 3)
    print(json.dumps({"catalog": cat, "elts": J, "hot_events": info.hot_events,
                      "entries_per_hot_event": round(info.entries / max(info.hot_events, 1), 2),
                      "ms_per_100k_trials": res, "lib": os.environ.get("ARE_LIB", "default")}), flush=True)
