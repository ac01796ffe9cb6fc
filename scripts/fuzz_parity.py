"""Randomised parity fuzz of every K2 path against the C oracle (test
infrastructure: the oracle is the checker).

Each case draws a catalog (tiny .. beyond twice the shared-memory filter), a
pool of ELTs with random sizes, explicit zero losses and random (sometimes
degenerate) financial terms, a ragged YET with empty trials, and 1-5 layers
with random occurrence / aggregate terms; then compares, bit for bit:
  * run_aggregate_analysis (auto kernel choice, fused layers when possible),
  * the same with EngineConfig(precombine=True),
  * price_layer per layer with the dense kernel,
  * a DeviceYearEventTable run, and the exact fused layer kernel on it,
against oracle.run_trials_port per layer; and K3 (PML exact, TVaR rel 1e-12)
plus the portfolio roll-up on every YLT.

    python scripts/fuzz_parity.py [--seconds 300] [--seed 1]
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1308_2066_b200.direct_access import TableSet  # noqa: E402
from paper_1308_2066_b200.engine import (EngineConfig, _fusable, layer_pool, price_layer,  # noqa: E402
                                         run_aggregate_analysis, simulate_layers_device)
from paper_1308_2066_b200.errors import PortfolioInvalidError  # noqa: E402
from paper_1308_2066_b200.portfolio import (EventLossTable, FinancialTerms, Layer, LayerTerms,  # noqa: E402
                                            YearEventTable)
from paper_1308_2066_b200.resident import DeviceYearEventTable  # noqa: E402
from paper_1308_2066_b200.risk import order_stats, portfolio_rollup  # noqa: E402


def want_ylt(layer, yet):
    stacked = oracle.dense_tables(layer.elts, yet.catalog_size)
    fin = [np.array([getattr(e.terms, f) for e in layer.elts], dtype=np.float64)
           for f in ("exchange_rate", "event_retention", "event_limit", "share")]
    t = layer.terms
    out = np.empty(yet.trial_count)
    oracle.run_trials_port(yet.event_ids, yet.offsets, stacked, np.arange(len(layer.elts), dtype=np.int64), *fin,
                           t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit, 0, 0, yet.trial_count, out)
    return out


def case(rng):
    cat = int(rng.choice([int(rng.integers(10, 3000)), int(rng.integers(3000, 300_000)),
                          int(rng.integers(1_600_000, 4_000_000))]))
    npool = int(rng.integers(1, 18))
    degenerate = rng.random() < 0.1
    pool = []
    for _ in range(npool):
        size = int(rng.integers(1, max(2, min(cat, 40_000))))
        ids = np.unique(rng.integers(1, cat + 1, size)).astype(np.uint32)
        loss = rng.lognormal(0, 1.2, ids.size) * 500.0
        loss[rng.random(ids.size) < 0.05] = 0.0
        terms = FinancialTerms(float(rng.uniform(0.3, 2.0)), float(rng.choice([0.0, rng.uniform(0, 400)])),
                               float(rng.choice([math.inf, rng.uniform(100, 5000)])), float(rng.uniform(0.05, 1.0)))
        pool.append(EventLossTable(cat, ids, loss, terms))
    nlay = int(rng.integers(1, 6))
    layers = []
    for i in range(nlay):
        k = int(rng.integers(1, npool + 1))
        sel = np.sort(rng.choice(npool, size=k, replace=False))
        lt = LayerTerms(float(rng.choice([0.0, rng.uniform(0, 600)])), float(rng.choice([math.inf, rng.uniform(50, 6000)])),
                        float(rng.choice([0.0, rng.uniform(0, 20_000)])),
                        float(rng.choice([math.inf, rng.uniform(100, 80_000)])))
        layers.append(Layer(f"L{i}", tuple(pool[j] for j in sel), lt))
    ntr = int(rng.integers(1, 3000))
    lens = rng.integers(1, int(rng.choice([60, 400, 2500])), ntr)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ids = rng.integers(1, cat + 1, int(offs[-1])).astype(np.uint32)
    yet = YearEventTable(cat, ids, None, offs)
    return pool, layers, yet, degenerate


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    n = 0
    while time.time() < t_end:
        pool, layers, yet, degenerate = case(rng)
        wants = [want_ylt(lay, yet) for lay in layers]
        for cfg in (EngineConfig(), EngineConfig(precombine=True)):
            got = run_aggregate_analysis(layers, yet, cfg)
            for lay, w, g in zip(layers, wants, got):
                assert g.losses.tobytes() == w.tobytes(), (n, lay.id, cfg)
        # K3 on every YLT and on the portfolio roll-up: PML exact, TVaR rel 1e-12
        ylts = list(got)
        roll = portfolio_rollup(ylts).losses
        want_roll = np.zeros(yet.trial_count)
        for w in wants:
            want_roll = want_roll + w  # list order, like metrics.py:118-133
        assert roll.tobytes() == want_roll.tobytes(), (n, "rollup")
        n_tr = yet.trial_count
        rps = [rp for rp in (1.5, 2.0, 10.0, 50.0, 100.0, 250.0, float(n_tr)) if 1.0 < rp <= n_tr]
        for w in wants + [want_roll]:
            if not rps:
                break
            p, t = order_stats(w, rps)
            for rp, pv, tv in zip(rps, p, t):
                assert pv == oracle.pml(w, rp), (n, "pml", rp)
                ref = oracle.tvar(w, rp)
                assert abs(tv - ref) <= 1e-12 * max(abs(ref), 1e-300) or (math.isnan(tv) and math.isnan(ref)), (n, "tvar")
        dyet = DeviceYearEventTable(yet)
        got = run_aggregate_analysis(layers, dyet)
        for w, g in zip(wants, got):
            assert g.losses.tobytes() == w.tobytes(), (n, "resident")
        if _fusable(layers, EngineConfig()) is not None:  # the exact fused kernel at any layer count
            pe, masks = layer_pool(layers)
            fz = simulate_layers_device(dyet, TableSet.from_elts(pe, yet.catalog_size), masks,
                                        [lay.terms for lay in layers]).cpu().numpy()
            for w, g in zip(wants, fz):
                assert g.tobytes() == w.tobytes(), (n, "fused")
        for lay, w in zip(layers, wants):
            ts = TableSet.from_elts(lay.elts, yet.catalog_size)
            terms = lay.terms
            if degenerate:  # terms the hot set cannot skip zeros for: AUTO runs the dense kernel
                terms = LayerTerms(-abs(terms.occ_retention) - 1.0, terms.occ_limit, terms.agg_retention, terms.agg_limit)
                lay2 = Layer(lay.id, lay.elts, terms)
                w = want_ylt(lay2, yet)
            g, _ = price_layer(yet, ts, None, terms, EngineConfig(variant="dense"))
            assert g.tobytes() == w.tobytes(), (n, lay.id, "dense")
            g, _ = price_layer(yet, ts, None, terms)
            assert g.tobytes() == w.tobytes(), (n, lay.id, "auto")
        n += 1
    print(f"fuzz ok: {n} random cases, every path bit-identical to the oracle")


if __name__ == "__main__":
    try:
        main()
    except PortfolioInvalidError as e:  # a generator bug, not a kernel one
        print("invalid case generated:", e)
        raise
