"""K2 time vs events per trial (C5 J=15 column) for the current build/env.

    python scripts/time_k2_e.py [--es 100,250,500,1000,2000] [--j 15]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from scripts.sweep import device_yet, time_k2, CATALOG
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.portfolio import LayerTerms
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt

ap = argparse.ArgumentParser()
ap.add_argument("--es", default="100,250,500,1000,2000")
ap.add_argument("--j", type=int, default=15)
args = ap.parse_args()
spec = GeneratorSpec(seed=2066, catalog_size=CATALOG, elt_count=args.j, elt_size_range=(10_000, 30_000))
tset = TableSet.from_elts([generate_elt(spec, i) for i in range(args.j)], CATALOG)
plan = tset.plan(*tset.selection_arrays(None))
terms = LayerTerms(500.0, 10_000.0, 140_000.0, 66_000.0)
tag = "stream" if os.environ.get("ARE_K2_STREAM") == "1" else "hotset"
for e in map(int, args.es.split(",")):
    t = int(1e9 // e)
    dyet = device_yet(t, e, seed=e)
    ms = time_k2(dyet, plan, terms)
    print(json.dumps({"kernel": tag, "events": e, "elts": args.j, "trials": t, "k2_ms": round(ms, 4),
                      "M_trials_per_s": round(t / ms / 1e3, 1)}), flush=True)
    del dyet
    torch.cuda.empty_cache()
from paper_1308_2066_b200 import _native  # noqa: E402
info = _native.plan_info(plan)
print(json.dumps({"plan": {"hot_events": info.hot_events, "filter_bits": info.filter_bits,
                           "smem_bytes": info.smem_bytes, "entries": info.entries}}))
