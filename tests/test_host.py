"""Host-side logic that needs no GPU: the partition, validation, config,
term helpers, footprint accounting, metric argument checks, and the C-ABI
library's exported surface."""

from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import BYTES_PER_SLOT, DirectAccessTable, memory_footprint
from paper_1308_2066_b200.engine import (
    EngineConfig,
    apply_aggregate_terms,
    apply_financial_terms,
    apply_occurrence_terms,
    resolve_backend,
    split_by_events,
)
from paper_1308_2066_b200.errors import EventOutOfRangeError, PortfolioInvalidError
from paper_1308_2066_b200.portfolio import (
    UNLIMITED,
    EventLossTable,
    FinancialTerms,
    Layer,
    LayerTerms,
    Trial,
    YearEventTable,
    validate_portfolio,
)
from paper_1308_2066_b200.risk import EPCurve, _order_stat_k
from tests.conftest import ROOT


# ------------------------------------------------------------- partition --

def test_split_by_events_matches_reference(golden):
    for case in golden["split_by_events"]:
        offs = np.zeros(len(case["lens"]) + 1, np.int64)
        np.cumsum(case["lens"], out=offs[1:])
        assert [list(b) for b in split_by_events(offs, case["parts"])] == case["batches"]


def test_split_covers_all_trials():
    offs = np.arange(0, 1001, 10, dtype=np.int64)
    for parts in (1, 2, 3, 8, 100, 500):
        b = split_by_events(offs, parts)
        assert b[0][0] == 0 and b[-1][1] == 100
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))


# ------------------------------------------------------------ validation --

def _layer(**kw):
    elt = EventLossTable.from_records({4: 100.0, 9: 50.0}, catalog_size=10, terms=kw.pop("fin", None))
    return Layer("L", (elt,), kw.pop("terms", LayerTerms()))


def _cats(layers, yet):
    return {v.category for v in validate_portfolio(layers, yet)}


def test_valid_portfolio_has_no_violations():
    yet = YearEventTable.from_trials([Trial.from_events([4, 9, 4])], catalog_size=10)
    assert validate_portfolio([_layer()], yet) == []


@pytest.mark.parametrize("case,category", [
    ("out_of_range", "event_out_of_range"),
    ("no_trials", "no_trials"),
    ("empty_trial", "trial_length"),
    ("bad_ts", "bad_timestamp"),
    ("unsorted", "trial_unsorted"),
    ("bad_fin", "bad_financial_terms"),
    ("bad_layer", "bad_layer_terms"),
    ("inf_retention", "bad_layer_terms"),
    ("no_elts", "layer_no_elts"),
    ("catalog", "catalog_mismatch"),
    ("negative_loss", "negative_loss"),
    ("duplicate", "duplicate_event"),
])
def test_violation_categories(case, category):
    layers = [_layer()]
    yet = YearEventTable.from_trials([Trial.from_events([4, 9])], catalog_size=10)
    if case == "out_of_range":
        yet = YearEventTable.from_trials([Trial.from_events([99])], catalog_size=10)
    elif case == "no_trials":
        yet = YearEventTable(10, np.zeros(0, np.uint32), np.zeros(0), np.zeros(1, np.int64))
    elif case == "empty_trial":
        yet = YearEventTable.from_trials([Trial.from_events([])], catalog_size=10)
    elif case == "bad_ts":
        yet = YearEventTable.from_trials([Trial.from_events([4], [1.5])], catalog_size=10)
    elif case == "unsorted":
        yet = YearEventTable.from_trials([Trial.from_events([4, 9], [0.5, 0.1])], catalog_size=10)
    elif case == "bad_fin":
        layers = [_layer(fin=FinancialTerms(exchange_rate=-1.0))]
    elif case == "bad_layer":
        layers = [_layer(terms=LayerTerms(occ_retention=-1.0))]
    elif case == "inf_retention":
        layers = [_layer(terms=LayerTerms(agg_retention=math.inf))]
    elif case == "no_elts":
        layers = [Layer("E", (), LayerTerms())]
    elif case == "catalog":
        layers = [Layer("C", (EventLossTable.from_records({1: 1.0}, catalog_size=11),), LayerTerms())]
    elif case == "negative_loss":
        layers = [Layer("N", (EventLossTable(10, np.array([1], np.uint32), np.array([-1.0])),), LayerTerms())]
    elif case == "duplicate":
        layers = [Layer("D", (EventLossTable(10, np.array([3, 3], np.uint32), np.array([1.0, 2.0])),), LayerTerms())]
    assert category in _cats(layers, yet)


def test_boundary_drops_are_not_unsorted():
    yet = YearEventTable.from_trials([Trial.from_events([4, 9], [0.2, 0.9]), Trial.from_events([4], [0.1])], 10)
    assert validate_portfolio([_layer()], yet) == []


def test_portfolio_invalid_error_carries_report():
    err = PortfolioInvalidError(validate_portfolio([_layer()], YearEventTable.from_trials(
        [Trial.from_events([99])], catalog_size=10)))
    assert isinstance(err, ValueError)
    assert any(v.category == "event_out_of_range" for v in err.violations)
    assert issubclass(EventOutOfRangeError, IndexError)


# ---------------------------------------------------------------- config --

def test_engine_config_validation():
    for bad in (dict(worker_count=0), dict(chunk_size=0), dict(deterministic=False),
                dict(backend="cuda"), dict(backend="python"), dict(variant="fast")):
        with pytest.raises(ValueError):
            EngineConfig(**bad)
    assert resolve_backend("auto") == resolve_backend("b200") == "b200"
    EngineConfig(worker_count=8, chunk_size=None, variant="dense")


# ----------------------------------------------------------------- terms --

def test_term_kats():
    assert apply_financial_terms(30.0, FinancialTerms(2.0, 10.0, 40.0, 0.5)) == 20.0
    assert apply_financial_terms(1e12, FinancialTerms(event_retention=1.0, event_limit=UNLIMITED)) == 1e12 - 1.0
    t = LayerTerms(occ_retention=10.0, occ_limit=60.0)
    assert [apply_occurrence_terms(x, t) for x in (100.0, 50.0, 5.0)] == [60.0, 40.0, 0.0]
    assert apply_aggregate_terms([30.0, 30.0, 30.0], LayerTerms(agg_retention=50.0, agg_limit=30.0)) == 30.0
    assert apply_aggregate_terms([], LayerTerms(agg_retention=5.0)) == 0.0


def test_aggregate_terms_telescope(rng):
    for _ in range(500):
        x = rng.lognormal(1.0, 2.0, int(rng.integers(0, 40)))
        t = LayerTerms(agg_retention=float(rng.uniform(0, 50)), agg_limit=float(rng.uniform(0, 500)))
        want = min(max(math.fsum(x) - t.agg_retention, 0.0), t.agg_limit)
        assert abs(apply_aggregate_terms(x, t) - want) <= 1e-9 * max(1.0, want)


# ------------------------------------------------------------- footprint --

def test_memory_footprint_kats():
    one = DirectAccessTable(1000, np.zeros(1001), FinancialTerms(), 1)
    assert memory_footprint([one]).total_bytes == 8_008
    many = [DirectAccessTable(2_000_000, None, FinancialTerms(), 1) for _ in range(15)]
    fp = memory_footprint(many)
    assert fp.payload_slots == 30_000_000 and fp.payload_bytes == 240_000_000
    assert fp.overhead_bytes == 15 * BYTES_PER_SLOT


# --------------------------------------------------------------- metrics --

def test_order_stat_rank_rule():
    assert _order_stat_k(1000, 100.0) == 990
    assert _order_stat_k(10, 3.0) == 7
    assert _order_stat_k(100, 100.0) == 99
    for bad in (1.0, 0.5, 101.0):
        with pytest.raises(ValueError):
            _order_stat_k(100, bad)


def test_ep_curve_invariants():
    with pytest.raises(ValueError):
        EPCurve(((100.0, 0.5), (90.0, 0.1)))
    with pytest.raises(ValueError):
        EPCurve(((10.0, 0.1), (20.0, 0.1)))
    with pytest.raises(ValueError):
        EPCurve(((10.0, 1.5),))
    c = EPCurve(((500.0, 0.5), (900.0, 0.1)))
    assert list(c) == [(500.0, 0.5), (900.0, 0.1)] and c.losses == (500.0, 900.0)


def test_ep_curve_array_constructor_matches_the_pairwise_checks(rng):
    """EPCurve._from_arrays (the device EP path) raises exactly what the
    reference's pairwise __post_init__ loop raises, first failure first."""
    cases = [([1.0, 2.0, 3.0], [0.5, 0.2, 0.1]), ([1.0, 0.5], [0.5, 0.4]), ([1.0, 2.0], [0.5, 0.5]),
             ([2.0, 1.0, 3.0], [0.5, 0.6, 0.1]), ([1.0, 2.0], [1.5, 0.4]), ([1.0, float("nan")], [0.5, 0.1]),
             ([1.0, 2.0], [0.5, float("nan")]), ([5.0], [0.25])]
    for _ in range(200):
        n = int(rng.integers(1, 6))
        cases.append((list(np.round(rng.normal(0, 1, n), 1)), list(np.round(rng.uniform(-0.2, 1.2, n), 1))))
    for loss, prob in cases:
        def run(f):
            try:
                return f().points
            except ValueError as e:
                return str(e)
        want = run(lambda: EPCurve(tuple(zip(loss, prob))))
        got = run(lambda: EPCurve._from_arrays(np.asarray(loss, float), np.asarray(prob, float)))
        assert got == want or (isinstance(got, tuple) and str(got) == str(want)), (loss, prob, got, want)


def test_return_period_checks_match_the_scalar_rule():
    from paper_1308_2066_b200.risk import _check_rps, _order_stat_k

    for rps in ([2.0, 10.0], [1.0], [0.5, 3.0], [5.0, 2e6], [float("nan")], [3.0, 1e6, 1.0]):
        arr = np.asarray(rps, dtype=np.float64)
        want = None
        for r in rps:
            try:
                _order_stat_k(1_000_000, r)
            except ValueError as e:
                want = str(e)
                break
        try:
            _check_rps(1_000_000, arr)
            got = None
        except ValueError as e:
            got = str(e)
        assert got == want, rps


# --------------------------------------------------------- the C-ABI .so --

def _declared_symbols() -> list[str]:
    with open(os.path.join(ROOT, "include", "aggrisk_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(are_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.SIGNATURES), "binding and header disagree"


def test_library_loads_and_reports_without_gpu():
    lib = _native.load()
    assert lib.are_version() == 1
    n = ctypes.c_int(-1)
    rc = lib.are_device_count(ctypes.byref(n))
    if rc != 0:  # no GPU here: the call fails loudly instead of pretending
        assert _native.last_error()
    assert _native.launch_count() >= 0


# ------------------------------------------------------- multi-layer pool --

def test_layer_pool_orders_and_masks():
    from paper_1308_2066_b200.engine import layer_pool

    a, b, c, d = (EventLossTable.from_records({i + 1: 1.0}, 10) for i in range(4))
    pool, masks = layer_pool([Layer("x", (a, c)), Layer("y", (b, c, d)), Layer("z", (a, b))])
    assert [pool.index(e) for e in (a, b, c, d)] == [0, 1, 2, 3]
    assert masks == [0b0101, 0b1110, 0b0011]
    # a layer that orders c before a conflicts with a layer ordering a before c
    assert layer_pool([Layer("x", (a, c)), Layer("y", (c, a))]) is None
    assert layer_pool([Layer("x", (a, a))]) is None


def test_entry_point_fusion_rule():
    """The entry point fuses layers only where the fused pass pays
    (engine.FUSE_*): enough layers for the trial count, a sparse pool, exact
    terms; pre-combination always fuses."""
    from paper_1308_2066_b200 import engine
    from paper_1308_2066_b200.engine import _fusable

    cat = 1_000
    rng = np.random.default_rng(3)
    pool = [EventLossTable(cat, np.sort(rng.choice(np.arange(1, cat + 1), 200, replace=False)).astype(np.uint32),
                           rng.lognormal(0, 1, 200)) for _ in range(8)]
    sparse = [Layer(f"s{i}", tuple(pool[:4]), LayerTerms(float(i), 1e6)) for i in range(6)]  # 0.8 entries/event
    dense = [Layer(f"d{i}", tuple(pool), LayerTerms(float(i), 1e6)) for i in range(6)]        # 1.6 entries/event
    cfg, pre = EngineConfig(), EngineConfig(precombine=True)
    big, small = 10 ** 9, 10 ** 6
    assert _fusable(sparse, cfg) is not None                     # no size information: fusable
    assert _fusable(sparse[:4], cfg, cat, big) is None           # < FUSE_MIN_LAYERS at scale
    assert _fusable(sparse[:4], cfg, cat, small) is not None     # small runs fuse from 3 layers
    assert _fusable(sparse[:2], cfg, cat, small) is None
    assert _fusable(sparse, cfg, cat, big) is not None
    assert _fusable(dense, cfg, cat, big) is not None            # 1.6 <= FUSE_MAX_ENTRIES_PER_EVENT
    assert _fusable(dense, cfg, cat // 2, big) is None           # 3.2 entries per catalog event
    assert _fusable(dense, pre, cat // 2, big) is not None       # explicit pre-combination
    assert _fusable(sparse[:2], pre, cat, big) is not None
    assert _fusable(sparse, EngineConfig(variant="dense"), cat, big) is None
    neg = sparse[:5] + [Layer("neg", tuple(pool[:4]), LayerTerms(-1.0, 1e6))]
    assert _fusable(neg, cfg, cat, big) is None                  # not zero-exact: layers run singly
    assert engine.FUSE_MIN_LAYERS_SMALL <= engine.FUSE_MIN_LAYERS


# ------------------------------------- validation pinned to the reference --

def test_validation_report_equals_reference_fixture():
    """Byte-equal `[category] message` lists against the reference's own
    validate_portfolio (model.py:360-404) on 169 cases: its per-category
    tests (pkg/tests/test_model.py:138-258), NaN timestamps, id 0, empty and
    over-long trials, boundary drops, combined faults and a seeded random mix
    (tests/golden/make_validation.py)."""
    from tests.validation_cases import build, load_cases

    cases = load_cases()
    assert len(cases) >= 150
    for case in cases:
        layers, yet = build(case)
        got = [str(v) for v in validate_portfolio(layers, yet)]
        assert got == case["report"], case["name"]


def test_group_shard_bounds_follow_the_reference_partition(golden):
    """The trial -> GPU cut points are split_by_events (engine/__init__.py:151-159)."""
    from paper_1308_2066_b200.group import shard_bounds

    for case in golden["split_by_events"]:
        offs = np.zeros(len(case["lens"]) + 1, np.int64)
        np.cumsum(case["lens"], out=offs[1:])
        b = shard_bounds(offs, case["parts"])
        assert b[0] == 0 and b[-1] == len(case["lens"]) and np.all(np.diff(b) > 0)
        assert [[int(x), int(y)] for x, y in zip(b[:-1], b[1:])] == case["batches"]


def test_group_devices_env(monkeypatch):
    from paper_1308_2066_b200 import group

    monkeypatch.setenv("ARE_GROUP_DEVICES", "0,0,1")
    assert group.devices_for(8) == (0, 0, 1)
    assert group.devices_for(2) == (0, 0)
