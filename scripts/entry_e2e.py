"""Wall time of the reference entry point run_aggregate_analysis on a C2-size
HOST year event table (ids + timestamps in host memory), with and without
the HBM promotion (engine.PROMOTE_MIN_OCC), cold and repeated (cached device copy).

    python scripts/entry_e2e.py [--trials N]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1308_2066_b200.engine as engine
from paper_1308_2066_b200.portfolio import YearEventTable

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=1_000_000)
args = ap.parse_args()
layer = bench.make_layer()
ids = bench.make_yet(0, args.trials, os.cpu_count() or 8)
ts = np.tile(np.linspace(0.0, 1.0, bench.EVENTS), args.trials)
yet = YearEventTable(bench.CATALOG, ids.event_ids, ts, ids.offsets)
res = {"trials": args.trials, "events": bench.EVENTS, "host_bytes": int(ids.event_ids.nbytes + ts.nbytes)}
engine.run_aggregate_analysis([layer], yet.head(1000))  # library / context warm-up
# hbm_promoted: a cold call (upload + K0 validation of ids and timestamps);
# hbm_promoted_repeat: the same YET again (its device copy is cached)
for name, thr in (("host_validate_and_stream", 1 << 62), ("hbm_promoted", engine.PROMOTE_MIN_OCC),
                  ("hbm_promoted_repeat", engine.PROMOTE_MIN_OCC)):
    engine.PROMOTE_MIN_OCC = thr
    runs = []
    for rep in range(3):
        if name != "hbm_promoted_repeat":
            engine._promoted.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ylts, stats = engine.run_aggregate_analysis_with_stats([layer], yet)
        torch.cuda.synchronize()
        runs.append((time.perf_counter() - t0, stats.sim_seconds, stats.build_seconds))
    best = min(runs)  # host stalls on the shared boxes move single runs by up to ~0.7 s
    res[name] = {"wall_s": best[0], "sim_s": best[1], "build_s": best[2],
                 "wall_s_runs": [round(r[0], 4) for r in runs],
                 "pml100": float(np.sort(ylts[0].losses)[-args.trials // 100])}
print(json.dumps(res))
