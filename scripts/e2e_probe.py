"""Diagnose the e2e (pinned host YET -> price_layer) step time on one GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import price_layer
from paper_1308_2066_b200.portfolio import YearEventTable

layer = bench.make_layer()
yet = bench.make_yet(0, bench.TRIALS_PER_GPU, os.cpu_count() or 8)
tset = TableSet.from_elts(layer.elts, bench.CATALOG)
with bench.GpuLocalCpus(0):
    pinned = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory()
    h_off = torch.from_numpy(np.ascontiguousarray(yet.offsets)).pin_memory()
hyet = YearEventTable(bench.CATALOG, pinned.numpy().view(np.uint32), None, h_off.numpy())
lib = _native.load()
print("pinned:", lib.are_host_is_pinned(pinned.data_ptr()), lib.are_host_is_pinned(h_off.data_ptr()),
      "affinity", sorted(os.sched_getaffinity(0))[:4], "...", len(os.sched_getaffinity(0)))
for i in range(8):
    t = time.perf_counter(); price_layer(hyet, tset, None, layer.terms); torch.cuda.synchronize()
    print(f"price_layer {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
d = torch.empty(pinned.numel(), dtype=torch.int32, device="cuda")
for i in range(3):
    t = time.perf_counter(); d.copy_(pinned, non_blocking=True); torch.cuda.synchronize()
    print(f"one 4 GB copy {1e3*(time.perf_counter()-t):.1f} ms")
s = torch.cuda.Stream()
for i in range(3):
    t = time.perf_counter()
    with torch.cuda.stream(s):
        for a in range(0, pinned.numel(), 32 << 20):
            d[a:a + (32 << 20)].copy_(pinned[a:a + (32 << 20)], non_blocking=True)
    s.synchronize()
    print(f"chunked 128 MB copies {1e3*(time.perf_counter()-t):.1f} ms")
for i in range(3):
    t = time.perf_counter(); price_layer(hyet, tset, None, layer.terms); torch.cuda.synchronize()
    print(f"price_layer {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
