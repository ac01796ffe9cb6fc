"""price_layer / run_trials on ordinary (pageable) numpy arrays vs pinned
ones, C2 shape: the drop-in seam's host-side data path.

    python scripts/host_path.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import price_layer
from paper_1308_2066_b200.portfolio import YearEventTable

layer = bench.make_layer()
yet = bench.make_yet(0, bench.TRIALS_PER_GPU, os.cpu_count() or 8)
tset = TableSet.from_elts(layer.elts, bench.CATALOG)
pinned = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory()
h_off = torch.from_numpy(np.ascontiguousarray(yet.offsets)).pin_memory()
cases = {"pageable": yet, "pinned": YearEventTable(bench.CATALOG, pinned.numpy().view(np.uint32), None, h_off.numpy())}
for name, y in cases.items():
    price_layer(y, tset, None, layer.terms)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        price_layer(y, tset, None, layer.terms)
        ts.append(time.perf_counter() - t0)
    print(f"{name}: median {1e3 * float(np.median(ts)):.1f} ms, min {1e3 * min(ts):.1f} ms per 1M trials x 1000 "
          f"({4e9 / min(ts) / 1e9:.1f} GB/s of ids)", flush=True)
