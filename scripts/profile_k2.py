"""Minimal driver for ncu: C2 setup (bench.py's data), then a few K2 launches.

    python scripts/profile_k2.py [--variant hotset|dense] [--launches N] [--trials T] [--events E]

--events changes the occurrences per trial (C5's short-trial points run
k2_pair below 320 occurrences per trial).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_2066_b200.direct_access import TableSet  # noqa: E402
from paper_1308_2066_b200.resident import DeviceYearEventTable  # noqa: E402
from paper_1308_2066_b200.risk import order_stats  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="hotset")
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--trials", type=int, default=bench.TRIALS_PER_GPU)
    ap.add_argument("--events", type=int, default=bench.EVENTS)
    ap.add_argument("--k3", action="store_true")
    ap.add_argument("--h2d", action="store_true", help="also time a pinned 4 GB H2D copy")
    args = ap.parse_args()
    layer = bench.make_layer()
    bench.EVENTS = args.events
    yet = bench.make_yet(0, args.trials, os.cpu_count() or 8)
    tset = TableSet.from_elts(layer.elts, bench.CATALOG)
    plan = tset.plan(*tset.selection_arrays(None))
    dyet = DeviceYearEventTable(yet)
    out = torch.empty(args.trials, dtype=torch.float64, device="cuda")
    for _ in range(args.launches):
        dyet.simulate_device(plan, layer.terms, out=out, variant=args.variant, check=False)
        if args.k3:
            order_stats(out, bench.RPS)
    torch.cuda.synchronize()
    if args.h2d:
        src = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory()
        dst = torch.empty_like(src, device="cuda")
        for _ in range(3):
            t0 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"pinned H2D {src.numel() * 4 / dt / 1e9:.1f} GB/s")
        from paper_1308_2066_b200 import _native
        print("library sees torch pinned memory as pinned:", _native.load().are_host_is_pinned(src.data_ptr()))


if __name__ == "__main__":
    main()
