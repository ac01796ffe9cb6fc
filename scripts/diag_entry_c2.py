import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_1308_2066_b200.engine as engine
from paper_1308_2066_b200.portfolio import YearEventTable
layer = bench.make_layer()
ids = bench.make_yet(0, 1_000_000, os.cpu_count() or 8)
ts = np.tile(np.linspace(0.0, 1.0, bench.EVENTS), 1_000_000)
yet = YearEventTable(bench.CATALOG, ids.event_ids, ts, ids.offsets)
engine.run_aggregate_analysis([layer], yet.head(1000))
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if rep == 2:
        pr = cProfile.Profile(); pr.enable()
    ylts, stats = engine.run_aggregate_analysis_with_stats([layer], yet)
    torch.cuda.synchronize()
    if rep == 2:
        pr.disable()
    print(rep, time.perf_counter() - t0, stats.sim_seconds, stats.build_seconds, len(engine._promoted), flush=True)
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
