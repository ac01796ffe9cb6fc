"""Session re-pricing (service.py:213-241 semantics) on the device."""

from __future__ import annotations

import math
import time

import numpy as np
import pytest

import oracle
from paper_1308_2066_b200.direct_access import build_count
from paper_1308_2066_b200.errors import PortfolioInvalidError
from paper_1308_2066_b200.portfolio import EventLossTable, LayerTerms, Trial, YearEventTable
from paper_1308_2066_b200.session import PricingSession
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def portfolio():
    spec = GeneratorSpec(seed=77, catalog_size=50_000, trial_count=50_000,
                         events_per_trial_range=(1000, 1000), elt_count=3, elt_size_range=(10_000, 30_000))
    return generate_yet(spec, ids_only=True), [generate_elt(spec, i) for i in range(3)]


def test_reprice_matches_reference_pipeline(portfolio):
    yet, elts = portfolio
    s = PricingSession(yet, elts)
    before = build_count()
    for terms, sel in [(LayerTerms(1000.0, 50_000.0, 0.0, math.inf), None),
                       (LayerTerms(500.0, 20_000.0, 100_000.0, 400_000.0), [2, 0]),
                       (LayerTerms(0.0, math.inf, 0.0, math.inf), [1])]:
        out = s.reprice(terms, sel, [10, 50, 100, 250, 50])
        picked = [elts[i] for i in (sel if sel is not None else range(3))]
        stacked = oracle.dense_tables(picked, yet.catalog_size)
        fin = [np.ones(len(picked)), np.zeros(len(picked)), np.full(len(picked), np.inf), np.ones(len(picked))]
        want, _ = oracle.run_layer_cpu(yet.event_ids, yet.offsets, stacked, fin,
                                       (terms.occ_retention, terms.occ_limit, terms.agg_retention,
                                        terms.agg_limit), workers=8, kernel="port")
        assert s.losses().tobytes() == want.tobytes()
        for m in out["metrics"]:
            assert m["pml"] == oracle.pml(want, m["return_period"])
            assert m["tvar"] == pytest.approx(oracle.tvar(want, m["return_period"]), rel=1e-12)
        assert [(p["loss"], p["exceedance_probability"]) for p in out["ep_curve"]] == \
            list(oracle.ep_points(want, [10, 50, 100, 250]))
        assert out["lookups"] == 50_000 * 1000 * len(picked)
        assert out["trial_max"] == want.max()
        assert out["trial_mean"] == pytest.approx(want.mean(), rel=1e-12)
    assert build_count() == before and s.reprice_count == 3


def test_interactive_latency(portfolio):
    """Reference acceptance: reprice of 50K x 1000 x 3 within 5 s (0.29 s recorded)."""
    yet, elts = portfolio
    s = PricingSession(yet, elts)
    s.reprice(LayerTerms(1000.0, 50_000.0))
    t0 = time.perf_counter()
    out = s.reprice(LayerTerms(1000.0, 50_000.0, 0.0, math.inf), None, [10, 50, 100, 250])
    wall = time.perf_counter() - t0
    assert wall < 0.05, wall
    print(f"reprice 50K x 1000 x 3: {wall * 1e3:.2f} ms wall ({out['engine_seconds'] * 1e3:.2f} ms engine)")


def test_invalid_session_and_bad_return_period():
    elt = EventLossTable.from_records({4: 1.0}, catalog_size=10)
    bad = YearEventTable.from_trials([Trial.from_events([11])], catalog_size=10)
    with pytest.raises(PortfolioInvalidError):
        PricingSession(bad, [elt])
    ok = YearEventTable.from_trials([Trial.from_events([4])] * 5, catalog_size=10)
    s = PricingSession(ok, [elt])
    with pytest.raises(ValueError):
        s.reprice(LayerTerms(), None, [6.0])
