"""Time the dense (uncompacted, event-major) K2 kernel on C2 data (CUDA events).

    python scripts/time_dense.py [--trials N] [--reps R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_2066_b200.direct_access import TableSet  # noqa: E402
from paper_1308_2066_b200.resident import DeviceYearEventTable  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
layer = bench.make_layer()
yet = bench.make_yet(0, args.trials, os.cpu_count() or 8)
tset = TableSet.from_elts(layer.elts, bench.CATALOG)
plan = tset.plan(*tset.selection_arrays(None))
dyet = DeviceYearEventTable(yet)
out = {v: torch.empty(args.trials, dtype=torch.float64, device="cuda") for v in ("dense", "hotset")}
for v in ("dense", "hotset"):
    for _ in range(2):
        dyet.simulate_device(plan, layer.terms, out=out[v], variant=v, check=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        dyet.simulate_device(plan, layer.terms, out=out[v], variant=v, check=False)
    b.record()
    torch.cuda.synchronize()
    print(f"K2 {v}: {a.elapsed_time(b) / args.reps:.3f} ms per {args.trials} trials "
          f"({os.environ.get('ARE_LIB', 'default build')})")
print("bitwise equal:", bool(torch.equal(out["dense"], out["hotset"])))
