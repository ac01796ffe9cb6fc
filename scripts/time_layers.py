"""Time the fused multi-layer kernel alone on the C3 shape (CUDA events).

    python scripts/time_layers.py [--trials N] [--reps R]
"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from scripts.sweep import device_yet, CATALOG
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import layer_pool, simulate_layers_device
from paper_1308_2066_b200.portfolio import Layer, LayerTerms
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_layer

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
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
pe, masks = layer_pool(layers)
ts = TableSet.from_elts(pe, CATALOG)
dyet = device_yet(args.trials, 1000, 33)
out = torch.empty((16, args.trials), dtype=torch.float64, device="cuda")
res = {}
for pre in (False, True):
    for _ in range(2):
        simulate_layers_device(dyet, ts, masks, [l.terms for l in layers], out=out, precombine=pre)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        simulate_layers_device(dyet, ts, masks, [l.terms for l in layers], out=out, precombine=pre)
    b.record()
    torch.cuda.synchronize()
    res[pre] = out.clone()
    print(f"fused 16-layer K2{' pre-combined' if pre else ''}: {a.elapsed_time(b) / args.reps:.3f} ms per "
          f"{args.trials} trials ({os.environ.get('ARE_LIB', 'default build')})")
print("bitwise equal:", bool(torch.equal(res[False], res[True])))
