"""K0 device validation and the direct ARE1 -> HBM loader, against the host
restatement of validate_portfolio (whose categories/messages mirror
model.py:360-404)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import price_layer, run_aggregate_analysis
from paper_1308_2066_b200.errors import PortfolioInvalidError
from paper_1308_2066_b200.portfolio import (
    EventLossTable,
    Layer,
    LayerTerms,
    Trial,
    YearEventTable,
    validate_portfolio,
)
from paper_1308_2066_b200.resident import DeviceYearEventTable
from paper_1308_2066_b200.yet_io import load_yet, load_yet_device, save_yet
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _layer(cat=50):
    return Layer("L", (EventLossTable.from_records({4: 100.0, 9: 50.0}, cat),), LayerTerms(1.0, 60.0, 5.0, 500.0))


def _yet(cases: str, cat=50):
    rng = np.random.default_rng(5)
    trials = [Trial.from_events(rng.integers(1, cat + 1, int(rng.integers(1, 40)))) for _ in range(30)]
    if "range" in cases:
        trials[3] = Trial.from_events([1, cat + 1, 2])
    if "zero_id" in cases:
        trials[4] = Trial.from_events([0, 3])
    if "empty" in cases:
        trials[7] = Trial.from_events([])
    if "long" in cases:
        trials[9] = Trial.from_events(np.ones(10_001, dtype=np.int64))
    if "ts_range" in cases:
        trials[2] = Trial.from_events([1, 2], [0.5, 1.5])
    if "unsorted" in cases:
        trials[5] = Trial.from_events([1, 2, 3], [0.1, 0.9, 0.2])
        trials[6] = Trial.from_events([1, 2], [0.8, 0.3])
    if "nan" in cases:
        trials[8] = Trial.from_events([1, 2], [np.nan, 2.0])  # numpy: NaN hides the range error
    return YearEventTable.from_trials(trials, cat)


@pytest.mark.parametrize("cases", ["", "range", "zero_id", "empty", "long", "ts_range", "unsorted",
                                   "nan", "range empty ts_range unsorted", "long unsorted zero_id"])
def test_device_report_matches_host_validation(cases):
    yet = _yet(cases)
    want = [str(v) for v in validate_portfolio([_layer()], yet)]
    dyet = DeviceYearEventTable(yet)
    got = [str(v) for v in validate_portfolio([_layer()], dyet)]
    assert got == want
    assert dyet.ids_validated == ("range" not in cases)


def test_chunked_timestamp_validation_counts_every_chunk():
    yet = _yet("unsorted ts_range")
    dyet = DeviceYearEventTable.from_host_arrays(yet.catalog_size, yet.event_ids, yet.offsets)
    dyet.validate_timestamps(yet.timestamps, chunk=17)  # many trial-aligned chunks
    assert [str(v) for v in dyet.yet_violations()] == \
        [str(v) for v in validate_portfolio([], yet) if v.category != "no_trials"]


def test_invalid_device_yet_refused_by_entry_point():
    with pytest.raises(PortfolioInvalidError):
        run_aggregate_analysis([_layer()], DeviceYearEventTable(_yet("range")))


def test_are1_straight_to_device_matches_host(tmp_path):
    path = os.path.join(GOLDEN, "yet_small.are1")
    host = load_yet(path)
    dyet = load_yet_device(path, chunk=1000)
    assert validate_portfolio([], dyet) == [v for v in validate_portfolio([], host)]
    rng = np.random.default_rng(1)
    elt = EventLossTable(host.catalog_size, np.sort(rng.choice(np.arange(1, host.catalog_size + 1), 400,
                                                               replace=False)).astype(np.uint32),
                         rng.lognormal(0, 1, 400) * 100)
    layer = Layer("x", (elt,), LayerTerms(10.0, 300.0, 50.0, 5000.0))
    tset = TableSet.from_elts(layer.elts, host.catalog_size)
    a, _ = price_layer(host, tset, None, layer.terms)
    b, _ = price_layer(dyet, tset, None, layer.terms)
    assert a.tobytes() == b.tobytes()
    # ids-only file: a bad timestamp written on disk is reported from the device scan
    bad = YearEventTable(host.catalog_size, host.event_ids, np.where(np.arange(host.event_ids.size) == 7, 3.0,
                                                                     host.timestamps), host.offsets)
    save_yet(bad, tmp_path / "bad.are1")
    cats = [v.category for v in load_yet_device(tmp_path / "bad.are1").yet_violations()]
    assert "bad_timestamp" in cats


@pytest.mark.parametrize("cases", ["", "range", "unsorted", "long unsorted zero_id", "nan"])
def test_entry_point_promotes_large_host_yets(monkeypatch, cases):
    """run_aggregate_analysis moves large host YETs into HBM (K0 validation,
    resident ids): same violations (as the exception's report) and the same
    bits as the host-validated, host-streamed path."""
    import paper_1308_2066_b200.engine as engine
    from paper_1308_2066_b200.engine import run_aggregate_analysis_with_stats

    yet = _yet(cases)
    layers = [_layer(), Layer("M", _layer().elts, LayerTerms(0.0, 70.0, 0.0, 300.0))]

    def run():
        try:
            return run_aggregate_analysis_with_stats(layers, yet)
        except PortfolioInvalidError as err:
            return [str(v) for v in err.violations]

    host = run()
    monkeypatch.setattr(engine, "PROMOTE_MIN_OCC", 1)
    dev = run()
    if isinstance(host, list):
        assert dev == host
        return
    (hy, hs), (dy, ds) = host, dev
    assert [y.losses.tobytes() for y in dy] == [y.losses.tobytes() for y in hy]
    assert (ds.trials, ds.layers, ds.lookups) == (hs.trials, hs.layers, hs.lookups)


def test_promoted_yet_is_cached_per_host_object(monkeypatch):
    """Repeated analyses of one large host YET upload and validate it once;
    the device copy goes when the host YET is collected, and it never keeps
    the host YET alive."""
    import gc

    import paper_1308_2066_b200.engine as engine

    monkeypatch.setattr(engine, "PROMOTE_MIN_OCC", 1)
    yet = _yet("")
    layers = [_layer()]
    first = engine.run_aggregate_analysis(layers, yet)
    d1 = engine._promote(yet)
    assert engine._promote(yet) is d1 and any(k[0] == id(yet) for k in engine._promoted)
    again = engine.run_aggregate_analysis(layers, yet)
    assert [y.losses.tobytes() for y in again] == [y.losses.tobytes() for y in first]
    assert d1.event_ids is yet.event_ids or np.array_equal(d1.event_ids, yet.event_ids)
    key = id(yet)
    del yet, d1
    gc.collect()
    assert all(k[0] != key for k in engine._promoted)
    bad = _yet("range")
    for _ in range(2):  # the cached copy keeps reporting the violation
        with pytest.raises(PortfolioInvalidError):
            engine.run_aggregate_analysis(layers, bad)


def test_k0_reports_equal_reference_fixture(tmp_path):
    """K0 (DeviceYearEventTable) and the ARE1 -> HBM loader produce the
    reference's own validate_portfolio report (model.py:360-404) byte for
    byte on the 169 reference-written cases (tests/golden/validation.json.gz,
    tests/golden/make_validation.py) -- not just the repo's host restatement."""
    from tests.validation_cases import build, load_cases

    for i, case in enumerate(load_cases()):
        layers, yet = build(case)
        dyet = DeviceYearEventTable(yet)
        got = [str(v) for v in validate_portfolio(layers, dyet)]
        assert got == case["report"], case["name"]
        if yet.offsets.size > 1 and i % 4 == 0:  # the direct file loader on a quarter of them
            path = tmp_path / f"c{i}.are1"
            save_yet(yet, path)
            got = [str(v) for v in validate_portfolio(layers, load_yet_device(path, chunk=7))]
            assert got == case["report"], case["name"] + " (ARE1)"
