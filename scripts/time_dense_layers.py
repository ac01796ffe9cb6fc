"""Multi-layer analyses in the dense-overlap regime (the reference's 50k
catalog): the fused hot-set layer kernel (K2-L) vs one event-major dense K2
per layer.  ms per 100k trials x 1000 events, CUDA events.

    python scripts/time_dense_layers.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import numpy as np
import torch
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import layer_pool, simulate_layers_device
from paper_1308_2066_b200.portfolio import Layer, LayerTerms
from paper_1308_2066_b200.resident import DeviceYearEventTable
from paper_1308_2066_b200.synth import GeneratorSpec, bulk_yet, generate_elt

T = 100_000
SHAPES = ((50_000, 15, 15), (50_000, 15, 8), (200_000, 32, 15), (200_000, 15, 15), (150_000, 15, 15),
          (120_000, 15, 15), (50_000, 3, 3))
if len(sys.argv) > 1:
    SHAPES = SHAPES[int(sys.argv[1]):]
for cat, P, per in SHAPES:
    spec = GeneratorSpec(seed=7, catalog_size=cat, elt_count=P, elt_size_range=(10_000, 30_000))
    pool = [generate_elt(spec, i) for i in range(P)]
    dyet = DeviceYearEventTable(bulk_yet(7, cat, 0, T, 1000, threads=8))
    rng = np.random.default_rng(1)
    for L in (2, 4, 8, 16):
        layers = [Layer(f"L{i}", tuple(pool[j] for j in np.sort(rng.choice(P, per, replace=False))),
                        LayerTerms(float(i * 10), 1e6, 0.0, float("inf"))) for i in range(L)]
        pe, masks = layer_pool(layers)
        ptset = TableSet.from_elts(pe, cat)
        terms = [l.terms for l in layers]
        fused = torch.empty((L, T), dtype=torch.float64, device="cuda")
        singles = [(TableSet.from_elts(l.elts, cat), l.terms) for l in layers]
        plans = [(ts.plan(*ts.selection_arrays(None)), t) for ts, t in singles]
        outs = [torch.empty(T, dtype=torch.float64, device="cuda") for _ in layers]

        def run_fused():
            simulate_layers_device(dyet, ptset, masks, terms, out=fused, check=False)

        def run_single():
            for (p, t), o in zip(plans, outs):
                dyet.simulate_device(p, t, out=o, check=False)

        res = {}
        for name, fn in (("fused_hotset", run_fused), ("per_layer_auto", run_single)):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[name] = round(a.elapsed_time(b) / 3, 3)
        same = all(torch.equal(fused[i], outs[i]) for i in range(L))
        dens = sum(len(e.event_ids) for e in pe) / cat
        print(json.dumps({"catalog": cat, "pool": P, "pool_entries_per_event": round(dens, 2), "elts_per_layer": per, "layers": L, "ms": res,
                          "bitwise_equal": same}), flush=True)
