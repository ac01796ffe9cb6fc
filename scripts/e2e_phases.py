"""Per-step, per-phase timing of bench.py's e2e path (pinned host YET ->
price_layer -> order_stats) to locate the occasional 0.1-1 s stalls.
    python scripts/e2e_phases.py [--steps 40] [--nvml]"""
import argparse, gc, json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import price_layer
from paper_1308_2066_b200.portfolio import YearEventTable
from paper_1308_2066_b200.risk import order_stats

ap = argparse.ArgumentParser(); ap.add_argument("--steps", type=int, default=40); ap.add_argument("--nvml", action="store_true")
ap.add_argument("--nogc", action="store_true")
args = ap.parse_args()
layer = bench.make_layer()
yet = bench.make_yet(0, bench.TRIALS_PER_GPU, os.cpu_count() or 8)
tset = TableSet.from_elts(layer.elts, bench.CATALOG)
with bench.GpuLocalCpus(0):
    pinned = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory()
    h_off = torch.from_numpy(np.ascontiguousarray(yet.offsets)).pin_memory()
hyet = YearEventTable(bench.CATALOG, pinned.numpy().view(np.uint32), None, h_off.numpy())
stop = threading.Event()
if args.nvml:
    import pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    def samp():
        while not stop.is_set():
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); pynvml.nvmlDeviceGetPowerUsage(h); time.sleep(0.01)
    threading.Thread(target=samp, daemon=True).start()
if args.nogc:
    gc.disable()
rows = []
for i in range(args.steps):
    t0 = time.perf_counter()
    ylt, _ = price_layer(hyet, tset, None, layer.terms)
    t1 = time.perf_counter()
    order_stats(ylt, bench.RPS)
    t2 = time.perf_counter()
    rows.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2)))
stop.set()
print(json.dumps({"nvml": args.nvml, "nogc": args.nogc, "price_ms": [r[0] for r in rows], "k3_ms": [r[1] for r in rows],
                  "median_price": float(np.median([r[0] for r in rows])), "max_price": max(r[0] for r in rows),
                  "max_k3": max(r[1] for r in rows)}))
