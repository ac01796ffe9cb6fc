"""K3 micro-benchmark: order_stats on 1M-trial YLTs of different shapes
(uniform, C2-like zeros + an atom at the aggregate limit, all-equal), timed
with CUDA events on the launching stream.  Prints one JSON line per case."""

from __future__ import annotations

import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import time  # noqa: E402

import numpy as np  # noqa: E402

from paper_1308_2066_b200.risk import ep_curve, order_stats, order_stats_summary, pml_many  # noqa: E402

RPS = [10.0, 50.0, 100.0, 250.0]


def cases(n: int):
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    yield "uniform", u * 1e5
    c2 = torch.where(u < 0.7, torch.zeros_like(u), torch.clamp((u - 0.7) * 3e5, max=66000.0))
    yield "c2_like", c2
    yield "all_equal", torch.full((n,), 5.0, device="cuda", dtype=torch.float64)
    yield "all_zero", torch.zeros(n, device="cuda", dtype=torch.float64)


def main() -> None:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    st = torch.cuda.current_stream()
    for name, x in cases(n):
        for _ in range(3):
            order_stats(x, RPS)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            pml, tvar = order_stats(x, RPS)
        e1.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"case": name, "n": n, "us_per_call": e0.elapsed_time(e1) * 1e3 / reps,
                          "pml": list(pml), "tvar": list(tvar)}))


def ep_timing(n: int) -> None:
    """A 100-point EP curve: one sort (pml_many) vs the select kernel in
    groups of 8 (order_stats), wall per call (both synchronise)."""
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 1e5
    rps = list(np.geomspace(1.01, n, 100))
    for name, fn in [("ep100_sort", lambda: pml_many(x, rps)), ("ep100_select", lambda: order_stats(x, rps)),
                     ("ep_curve_100", lambda: ep_curve(x, rps)),
                     ("summary_4rp_mean_max", lambda: order_stats_summary(x, RPS))]:
        for _ in range(3):
            fn()
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        print(json.dumps({"case": name, "n": n, "us_per_call_wall": (time.perf_counter() - t0) * 1e6 / reps}))


if __name__ == "__main__":
    main()
    ep_timing(int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000)
