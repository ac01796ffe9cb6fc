"""GPU parity: the CUDA path through the C-ABI against the reference's outputs.

Bar: the Year Loss Table is BIT-IDENTICAL to the reference CPU kernel
(_kernel.pyx) on the same inputs -- both K2 variants reproduce its float64
operation order exactly -- which is stricter than the
north-star tolerance |got - ref| <= 1e-5 * (|ref| + agg_retention).  PML is
an order statistic of identical data, hence also exact; TVaR is a mean whose
summation order differs from numpy's pairwise sum: rel 1e-12.
"""

from __future__ import annotations

import hashlib
import math
import os

import numpy as np
import pytest

import oracle
from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import TableSet, build_count, build_direct_table
from paper_1308_2066_b200.engine import (
    EngineConfig,
    analyse_trial,
    price_layer,
    run_aggregate_analysis,
    run_aggregate_analysis_with_stats,
    run_chunked,
    run_trials,
)
from paper_1308_2066_b200.errors import EventOutOfRangeError, PortfolioInvalidError
from paper_1308_2066_b200.portfolio import (
    EventLossTable,
    FinancialTerms,
    Layer,
    LayerTerms,
    Trial,
    YearEventTable,
)
from paper_1308_2066_b200.synth import GeneratorSpec, bulk_yet, generate_elt, generate_layer, generate_yet
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

HOT = EngineConfig(variant="hotset")
DENSE = EngineConfig(variant="dense")


def _worked():
    elt = EventLossTable.from_records({4: 100.0, 9: 50.0}, catalog_size=10)
    return Layer("L", (elt,), LayerTerms(10.0, 60.0, 0.0, 150.0)), Trial.from_events([4, 9, 4])


def _oracle_ylt(layer, yet, stacked=None, terms=None):
    stacked = oracle.dense_tables(layer.elts, yet.catalog_size) if stacked is None else stacked
    t = layer.terms if terms is None else terms
    fin = [np.array([getattr(e.terms, f) for e in layer.elts], dtype=np.float64)
           for f in ("exchange_rate", "event_retention", "event_limit", "share")]
    out = np.empty(yet.trial_count)
    oracle.run_trials_port(yet.event_ids, yet.offsets, stacked, np.arange(len(layer.elts), dtype=np.int64),
                           *fin, t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit,
                           0, 0, yet.trial_count, out)
    return out


# ------------------------------------------------------------ KATs -------

def test_worked_example():
    layer, trial = _worked()
    assert analyse_trial(trial, layer) == 150.0
    assert analyse_trial(trial, layer, TableSet.from_elts(layer.elts)) == 150.0
    assert analyse_trial(trial, layer, [build_direct_table(e) for e in layer.elts]) == 150.0
    assert analyse_trial(trial, layer, cfg=DENSE) == 150.0


def test_empty_trial_and_misaligned_tables():
    layer, _ = _worked()
    assert analyse_trial(Trial.from_events([]), layer) == 0.0
    other = build_direct_table(EventLossTable.from_records({1: 1.0}, catalog_size=10))
    with pytest.raises(ValueError):
        analyse_trial(Trial.from_events([4]), layer, [other, other])
    with pytest.raises(EventOutOfRangeError):
        analyse_trial(Trial.from_events([11]), layer)


def test_multi_layer_order_and_lookups(golden):
    elt = EventLossTable.from_records({1: 10.0}, catalog_size=5)
    layers = [Layer("first", (elt,), LayerTerms()), Layer("second", (elt,), LayerTerms(occ_limit=4.0))]
    yet = YearEventTable.from_trials([Trial.from_events([1])], catalog_size=5)
    ylts = run_aggregate_analysis(layers, yet)
    assert [y.layer_id for y in ylts] == ["first", "second"]
    assert [float(y.losses[0]) for y in ylts] == golden["kats"]["multi_layer"] == [10.0, 4.0]
    three = Layer("c", (elt, elt, elt), LayerTerms())
    yet7 = YearEventTable.from_trials([Trial.from_events([1, 2, 3, 4]) for _ in range(7)], catalog_size=5)
    _, stats = run_aggregate_analysis_with_stats([three], yet7)
    assert stats.lookups == 7 * 4 * 3 and stats.trials == 7 and stats.layers == 1
    with pytest.raises(ValueError):
        run_chunked([layers[0]], yet, EngineConfig(chunk_size=None))


def test_invalid_portfolio_refused():
    layer, _ = _worked()
    with pytest.raises(PortfolioInvalidError):
        run_aggregate_analysis([layer], YearEventTable.from_trials([Trial.from_events([99])], catalog_size=10))


# ---------------------------------------------- 1000 reference instances --

@pytest.mark.parametrize("cfg", [HOT, DENSE], ids=["hotset", "dense"])
def test_random_instances_bitwise_vs_reference(instances, cfg):
    for inst in instances:
        got = run_aggregate_analysis([inst.layer], inst.yet, cfg)[0].losses
        assert got.tobytes() == inst.ylt.tobytes()


def test_plugin_run_trials_bitwise(instances):
    """The reference seam: run_trials(...) with the reference's argument list."""
    for inst in instances[:300]:
        out = np.full(inst.yet.trial_count, -1.0)
        rows = np.arange(len(inst.layer.elts), dtype=np.int64)
        t = inst.layer.terms
        n = run_trials(inst.yet.event_ids, inst.yet.offsets, inst.stacked, rows, *inst.fin(),
                       t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit, 4,
                       0, inst.yet.trial_count, out, np.empty(4))
        assert out.tobytes() == inst.ylt.tobytes()
        assert n == len(rows) * int(inst.yet.offsets[-1])


def test_plugin_partial_range_and_arg_errors(instances):
    inst = max(instances, key=lambda i: i.yet.trial_count)
    n = inst.yet.trial_count
    rows = np.arange(len(inst.layer.elts), dtype=np.int64)
    t = inst.layer.terms
    args = (t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit)
    out = np.full(n, -7.0)
    a, b = n // 3, 2 * n // 3
    run_trials(inst.yet.event_ids, inst.yet.offsets, inst.stacked, rows, *inst.fin(), *args, 0, a, b, out, None)
    assert out[a:b].tobytes() == inst.ylt[a:b].tobytes()
    assert np.all(out[:a] == -7.0) and np.all(out[b:] == -7.0)
    with pytest.raises(ValueError):  # scratch < chunk
        run_trials(inst.yet.event_ids, inst.yet.offsets, inst.stacked, rows, *inst.fin(), *args, 4, 0, n, out,
                   np.empty(2))
    with pytest.raises(ValueError):  # wrong dtype
        run_trials(inst.yet.event_ids.astype(np.int64), inst.yet.offsets, inst.stacked, rows, *inst.fin(),
                   *args, 0, 0, n, out, None)
    with pytest.raises(ValueError):  # more than 256 tables
        run_trials(inst.yet.event_ids, inst.yet.offsets, inst.stacked, np.zeros(257, np.int64),
                   *(np.ones(257) for _ in range(4)), *args, 0, 0, n, out, None)


# ------------------------------------------------------ reference digests --

def test_seed31_digest_matches_reference(golden):
    """test_acceptance.py:93-118: generator + engine sha256 5ebdd83b8ee0."""
    spec = GeneratorSpec(seed=31, catalog_size=2_000, trial_count=10_000,
                         events_per_trial_range=(10, 50), elt_count=3, elt_size_range=(200, 800))
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(3)]
    layer = Layer("det", tuple(elts), LayerTerms(500.0, 20_000.0, 0.0, 300_000.0))
    for cfg in (HOT, DENSE, EngineConfig(worker_count=8, chunk_size=None)):
        ylt = run_aggregate_analysis([layer], yet, cfg)[0].losses
        assert hashlib.sha256(ylt.tobytes()).hexdigest() == golden["seed31"]["ylt_sha256"]
    assert golden["seed31"]["ylt_sha256"].startswith("5ebdd83b8ee0")


@pytest.fixture(scope="module")
def c1():
    spec = GeneratorSpec(seed=2066, catalog_size=2_000_000, trial_count=10_000,
                         events_per_trial_range=(1000, 1000), elt_count=15,
                         elt_size_range=(10_000, 30_000), loss_scale=1000.0)
    yet = generate_yet(spec, ids_only=True)
    elts = [generate_elt(spec, i) for i in range(15)]
    gen = generate_layer(spec, 0, elts)
    layer = Layer(gen.id, gen.elts, LayerTerms(500.0, 10_000.0, 140_000.0, 66_000.0))
    return yet, layer


def test_c1_ylt_bitwise_and_metrics(c1, golden):
    """10k x 1000 x 15 ELTs, catalog 2M, Cat XL + Agg XL."""
    from paper_1308_2066_b200.risk import order_stats

    yet, layer = c1
    ref = np.load(os.path.join(GOLDEN, "c1_ylt.npy"))
    tset = TableSet.from_elts(layer.elts, yet.catalog_size)
    for cfg in (HOT, DENSE):
        got, lookups = price_layer(yet, tset, None, layer.terms, cfg)
        assert got.tobytes() == ref.tobytes()
        assert lookups == 10_000 * 1000 * 15
    # north-star tolerance, stated for the record (exact equality implies it)
    assert np.all(np.abs(got - ref) <= 1e-5 * (np.abs(ref) + layer.terms.agg_retention))
    p, t = order_stats(got, golden["c1"]["rps"])
    assert list(p) == golden["c1"]["pml"]
    np.testing.assert_allclose(t, golden["c1"]["tvar"], rtol=1e-12)
    info = _native.plan_info(tset.plan(*tset.selection_arrays(None)))
    assert info.zero_skip_exact == 1 and info.hot_events > 0


def test_reprice_never_rebuilds_and_subset_selection(c1):
    yet, layer = c1
    small = yet.head(500)
    tset = TableSet.from_elts(layer.elts, yet.catalog_size)
    before = build_count()
    for k in range(5):
        terms = LayerTerms(500.0 * k, 10_000.0, 1000.0 * k, 50_000.0 + k)
        got, _ = price_layer(small, tset, None, terms)
        assert got.tobytes() == _oracle_ylt(layer, small, terms=terms).tobytes()
    assert build_count() == before
    picked = [14, 0, 7]  # arbitrary order = accumulation order
    got, n = price_layer(small, tset, picked, layer.terms)
    sub = Layer("sub", tuple(layer.elts[i] for i in picked), layer.terms)
    assert got.tobytes() == _oracle_ylt(sub, small).tobytes()
    assert n == 3 * int(small.offsets[-1])


# ------------------------------------------------------------ edge cases --

def test_degenerate_terms_fall_back_to_dense_exactly(instances):
    """Negative retentions make zero losses contribute (fin(0) != 0): the
    hot-set precondition fails, AUTO picks the dense kernel, still exact."""
    inst = instances[7]
    elts = tuple(EventLossTable(e.catalog_size, e.event_ids, e.losses, FinancialTerms(1.5, -3.0, 50.0, 0.5))
                 for e in inst.layer.elts)
    layer = Layer("neg", elts, LayerTerms(-2.0, 100.0, 5.0, 1000.0))
    tset = TableSet.from_elts(layer.elts, inst.yet.catalog_size)
    got, _ = price_layer(inst.yet, tset, None, layer.terms)
    assert got.tobytes() == _oracle_ylt(layer, inst.yet).tobytes()
    with pytest.raises(ValueError):
        price_layer(inst.yet, tset, None, layer.terms, HOT)


def test_nan_inf_and_zero_losses_flow_like_reference():
    cat = 50
    rng = np.random.default_rng(3)
    losses = rng.lognormal(0, 1, 20) * 10
    losses[:3] = [np.nan, np.inf, 0.0]
    elt = EventLossTable(cat, np.sort(rng.choice(np.arange(1, cat + 1), 20, replace=False)).astype(np.uint32),
                         losses, FinancialTerms(2.0, 1.0, np.inf, 0.75))
    elt2 = EventLossTable.from_records({1: 5.0, 2: 7.0, 3: 0.0}, cat, FinancialTerms(share=0.0))
    layer = Layer("x", (elt, elt2), LayerTerms(3.0, 40.0, 10.0, np.inf))
    yet = YearEventTable.from_trials([Trial.from_events(rng.integers(1, cat + 1, 37)) for _ in range(64)], cat)
    tset = TableSet.from_elts(layer.elts, cat)
    want = _oracle_ylt(layer, yet)
    assert np.isnan(want).any() and np.isinf(losses).any()
    for cfg in (HOT, DENSE):
        got, _ = price_layer(yet, tset, None, layer.terms, cfg)
        # NaN payloads are not portable (the GPU emits the canonical NaN);
        # every non-NaN value must match bitwise, NaNs must sit in the same trials
        assert np.array_equal(np.isnan(got), np.isnan(want))
        ok = ~np.isnan(want)
        assert got[ok].tobytes() == want[ok].tobytes()


@pytest.mark.parametrize("catalog", [1_700_000, 3_000_000, 9_000_000])
def test_large_catalogs_use_wrapped_filter_exactly(catalog):
    """Catalogs beyond the shared-memory filter (hash modes 1 and 2)."""
    rng = np.random.default_rng(catalog)
    elts = []
    for j in range(3):
        ids = np.unique(rng.integers(1, catalog + 1, 40_000)).astype(np.uint32)
        elts.append(EventLossTable(catalog, ids, rng.lognormal(0, 1, ids.size) * 100.0))
    layer = Layer("big", tuple(elts), LayerTerms(20.0, 500.0, 100.0, 5_000.0))
    trials = [Trial.from_events(np.concatenate([rng.integers(1, catalog + 1, 300),
                                                rng.choice(elts[0].event_ids, 30)])) for _ in range(200)]
    yet = YearEventTable.from_trials(trials, catalog)
    got = run_aggregate_analysis([layer], yet, HOT)[0].losses
    assert got.tobytes() == _oracle_ylt(layer, yet).tobytes()
    assert np.count_nonzero(got) > 0


@pytest.mark.parametrize("catalog", [50_000, 1_700_000, 3_000_000, 9_000_000])
def test_kernel_instantiations_across_hash_modes(catalog):
    """Every hot-set instantiation against the reference loop: filter hash
    mode 0/1/2 (catalog below, within 2x, beyond 2x the shared-memory bits),
    range-checked ids (price_layer: no validation) and validated ids (the
    entry point), per-table and pre-combined records, and the fused layer
    kernel on the same catalog."""
    rng = np.random.default_rng(catalog + 1)
    elts = []
    for j in range(4):
        ids = np.unique(rng.integers(1, catalog + 1, min(30_000, catalog // 3))).astype(np.uint32)
        terms = FinancialTerms(float(rng.uniform(0.8, 1.5)), float(rng.uniform(0, 50)), float(rng.uniform(500, 4000)),
                               float(rng.uniform(0.3, 1.0)))
        elts.append(EventLossTable(catalog, ids, rng.lognormal(0, 1, ids.size) * 300.0, terms))
    layer = Layer("L", tuple(elts), LayerTerms(30.0, 2_500.0, 800.0, 40_000.0))
    hot = np.concatenate([e.event_ids for e in elts])
    trials = [Trial.from_events(np.concatenate([rng.integers(1, catalog + 1, int(rng.integers(1, 600))),
                                                rng.choice(hot, int(rng.integers(0, 60)))])) for _ in range(300)]
    yet = YearEventTable.from_trials(trials, catalog)
    want = _oracle_ylt(layer, yet)
    assert np.count_nonzero(want) > 0
    tset = TableSet.from_elts(elts, catalog)
    for cfg in (HOT, EngineConfig(variant="hotset", precombine=True), DENSE):
        got, _ = price_layer(yet, tset, None, layer.terms, cfg)
        assert got.tobytes() == want.tobytes()
        assert run_aggregate_analysis([layer], yet, cfg)[0].losses.tobytes() == want.tobytes()
    # the dense kernel on an odd selection in non-pool order: with >= 64 MB of
    # selected rows (catalogs 3M, 9M) it reads the event-major copy
    sub = Layer("S", (elts[3], elts[0], elts[2]), layer.terms)
    got, _ = price_layer(yet, tset, [3, 0, 2], layer.terms, DENSE)
    assert got.tobytes() == _oracle_ylt(sub, yet).tobytes()
    second = Layer("M", tuple(elts[1:3]), LayerTerms(0.0, math.inf, 300.0, 20_000.0))
    want2 = _oracle_ylt(second, yet).tobytes()
    both = run_aggregate_analysis([layer, second], yet)  # two layers: run singly (FUSE_MIN_LAYERS)
    assert both[0].losses.tobytes() == want.tobytes() and both[1].losses.tobytes() == want2
    from paper_1308_2066_b200.engine import layer_pool, simulate_layers_device
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    pe, masks = layer_pool([layer, second])
    fused = simulate_layers_device(DeviceYearEventTable(yet), TableSet.from_elts(pe, catalog), masks,
                                   [layer.terms, second.terms]).cpu().numpy()
    assert fused[0].tobytes() == want.tobytes() and fused[1].tobytes() == want2


def test_256_tables_and_overflow_chains():
    cat = 300
    rng = np.random.default_rng(256)
    elts = tuple(EventLossTable(cat, np.sort(rng.choice(np.arange(1, cat + 1), 40, replace=False)).astype(np.uint32),
                                rng.lognormal(0, 1, 40), FinancialTerms(1.0, 0.1, 5.0, 0.9)) for _ in range(256))
    layer = Layer("wide", elts, LayerTerms(1.0, 200.0, 10.0, 2000.0))
    yet = YearEventTable.from_trials([Trial.from_events(rng.integers(1, cat + 1, 200)) for _ in range(40)], cat)
    for cfg in (HOT, DENSE):
        got = run_aggregate_analysis([layer], yet, cfg)[0].losses
        assert got.tobytes() == _oracle_ylt(layer, yet).tobytes()


def test_long_and_ragged_trials():
    cat = 5_000
    rng = np.random.default_rng(11)
    elt = EventLossTable(cat, np.arange(1, cat + 1, 3, dtype=np.uint32), rng.lognormal(0, 1, (cat + 2) // 3) * 50)
    layer = Layer("r", (elt,), LayerTerms(10.0, 300.0, 500.0, 1e6))
    lens = [0, 1, 2, 3, 4, 5, 31, 32, 33, 127, 128, 129, 130, 1000, 4099, 10_000, 7, 0]
    yet = YearEventTable(cat, rng.integers(1, cat + 1, sum(lens)).astype(np.uint32), None,
                         np.concatenate([[0], np.cumsum(lens)]).astype(np.int64))
    tset = TableSet.from_elts(layer.elts, cat)
    for cfg in (HOT, DENSE):
        got, _ = price_layer(yet, tset, None, layer.terms, cfg)
        assert got.tobytes() == _oracle_ylt(layer, yet).tobytes()
    # misaligned starts: every suffix of the occurrence stream
    for shift in range(1, 4):
        sub = YearEventTable(cat, yet.event_ids[shift:shift + 2500], None, np.array([0, 900, 2500], np.int64))
        got, _ = price_layer(sub, tset, None, layer.terms)
        assert got.tobytes() == _oracle_ylt(layer, sub).tobytes()


@pytest.mark.parametrize("n_sel", [4, 5, 15, 16, 17, 31, 32])
def test_dense_overlap_plans_event_major_kernel(n_sel):
    """Dense-overlap plans (several entries per catalog event: the reference's
    own bench shape) run the cooperative event-major dense kernel under AUTO;
    one and two line passes, odd selections (a padded slot), ragged trials and
    non-identity financial terms, all bitwise equal to the reference loop."""
    cat = 1_000
    rng = np.random.default_rng(n_sel)
    elts = tuple(EventLossTable(cat, np.sort(rng.choice(np.arange(1, cat + 1), 400, replace=False)).astype(np.uint32),
                                rng.lognormal(0, 1, 400) * 100,
                                FinancialTerms(float(rng.uniform(0.5, 1.5)), float(rng.uniform(0, 20)),
                                               float(rng.choice([math.inf, 150.0])), float(rng.uniform(0.2, 1.0))))
                 for _ in range(n_sel))
    layer = Layer("dense", elts, LayerTerms(30.0, 2_000.0, 100.0, 50_000.0))
    lens = rng.integers(0, 300, 200)
    lens[:6] = [0, 1, 31, 32, 33, 64]
    yet = YearEventTable(cat, rng.integers(1, cat + 1, int(lens.sum())).astype(np.uint32), None,
                         np.concatenate([[0], np.cumsum(lens)]).astype(np.int64))
    want = _oracle_ylt(layer, yet).tobytes()
    tset = TableSet.from_elts(layer.elts, cat)
    for cfg in (EngineConfig(), HOT, DENSE):
        got, _ = price_layer(yet, tset, None, layer.terms, cfg)
        assert got.tobytes() == want, cfg
    bad = YearEventTable(cat, np.array([4, cat + 1, 9], np.uint32), None, np.array([0, 3], np.int64))
    with pytest.raises(EventOutOfRangeError):
        price_layer(bad, tset, None, layer.terms, DENSE)


def test_loss_in_unused_slot_zero_is_honoured():
    """A dense table with a loss in column 0 (the reference reads it for event
    id 0) routes to the dense kernel and still matches the reference loop."""
    stacked = np.zeros((2, 11))
    stacked[0, 0], stacked[0, 4], stacked[1, 9] = 5.0, 100.0, 50.0
    ids = np.array([4, 0, 9, 0, 4], np.uint32)
    offs = np.array([0, 2, 5], np.int64)
    rows = np.arange(2, dtype=np.int64)
    fin = (np.ones(2), np.zeros(2), np.full(2, np.inf), np.ones(2))
    got, want = np.empty(2), np.empty(2)
    run_trials(ids, offs, stacked, rows, *fin, 1.0, 60.0, 0.0, 150.0, 0, 0, 2, got, None)
    oracle.run_trials_port(ids, offs, stacked, rows, *fin, 1.0, 60.0, 0.0, 150.0, 0, 0, 2, want)
    assert got.tobytes() == want.tobytes() and want[0] == 60.0 + 4.0


def test_event_out_of_range_in_yet_raises():
    layer, _ = _worked()
    yet = YearEventTable(10, np.array([4, 12, 9], np.uint32), None, np.array([0, 3], np.int64))
    tset = TableSet.from_elts(layer.elts, 10)
    with pytest.raises(EventOutOfRangeError):
        price_layer(yet, tset, None, layer.terms)


# -------------------------------------------------------- resident / pinned --

def test_resident_and_pinned_paths_match_host_path(c1):
    import torch

    from paper_1308_2066_b200.resident import DeviceYearEventTable

    yet, layer = c1
    tset = TableSet.from_elts(layer.elts, yet.catalog_size)
    ref = np.load(os.path.join(GOLDEN, "c1_ylt.npy"))
    dyet = DeviceYearEventTable(yet)
    got, n = price_layer(dyet, tset, None, layer.terms)
    assert got.tobytes() == ref.tobytes() and n == 15 * 10_000_000
    plan = tset.plan(*tset.selection_arrays(None))
    d = dyet.simulate_device(plan, layer.terms, 2000, 7000)
    assert d[2000:7000].cpu().numpy().tobytes() == ref[2000:7000].tobytes()
    pinned = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory().numpy().view(np.uint32)
    pyet = YearEventTable(yet.catalog_size, pinned, None, yet.offsets)
    got, _ = price_layer(pyet, tset, None, layer.terms)
    assert got.tobytes() == ref.tobytes()
    # pageable numpy ids (40 MB): staged into the pinned buffers by several threads
    got, _ = price_layer(yet, tset, None, layer.terms)
    assert got.tobytes() == ref.tobytes()


# ------------------------------------------ full-size properties (C2 shape) --

def test_c2_shape_sample_and_partition_invariance():
    """1M-trial shape, checked through size-independent properties: a random
    sample of trials equals the oracle exactly, and simulating the trials in
    shards (the multi-GPU partition) reproduces the whole YLT bit for bit."""
    from paper_1308_2066_b200.distributed import partition

    spec = GeneratorSpec(seed=2066, catalog_size=2_000_000, elt_count=15,
                         elt_size_range=(10_000, 30_000), loss_scale=1000.0)
    elts = [generate_elt(spec, i) for i in range(15)]
    layer = Layer("c2", tuple(elts), LayerTerms(500.0, 10_000.0, 140_000.0, 66_000.0))
    yet = bulk_yet(2066, 2_000_000, 0, 1_000_000, 1000, threads=16)
    tset = TableSet.from_elts(layer.elts, yet.catalog_size)
    whole, _ = price_layer(yet, tset, None, layer.terms)
    again, _ = price_layer(yet, tset, None, layer.terms)
    assert whole.tobytes() == again.tobytes()
    stacked = oracle.dense_tables(elts, yet.catalog_size)
    idx = np.random.default_rng(0).choice(yet.trial_count, 400, replace=False)
    for t in idx:
        a, b = int(yet.offsets[t]), int(yet.offsets[t + 1])
        one = YearEventTable(yet.catalog_size, yet.event_ids[a:b], None, np.array([0, b - a], np.int64))
        assert _oracle_ylt(layer, one, stacked)[0] == whole[t]
    for world in (2, 8):
        parts = partition(yet.offsets, world)
        pieces = []
        for a, b in parts:
            sub = YearEventTable(yet.catalog_size, yet.event_ids[yet.offsets[a]:yet.offsets[b]], None,
                                 yet.offsets[a:b + 1] - yet.offsets[a])
            pieces.append(price_layer(sub, tset, None, layer.terms)[0])
        assert np.concatenate(pieces).tobytes() == whole.tobytes()


# ------------------------------------------------- fused multi-layer (C3) --

def test_fused_layers_bitwise_equal_single_layer_runs():
    """one pass for 16 layers == 16 single-layer runs, bitwise."""
    import math as _m

    from paper_1308_2066_b200.engine import _fusable

    spec = GeneratorSpec(seed=2066, catalog_size=300_000, trial_count=3_000, events_per_trial_range=(200, 1200),
                         elt_count=32, elt_size_range=(2_000, 8_000), layer_count=16, elts_per_layer=15)
    yet = generate_yet(spec, ids_only=True)
    pool = [generate_elt(spec, i) for i in range(32)]
    from paper_1308_2066_b200.synth import generate_layer as _gl

    layers = []
    for i in range(16):
        g = _gl(spec, i, pool)
        t = g.terms
        terms = LayerTerms(t.occ_retention, t.occ_limit, 0.0, _m.inf) if i % 2 == 0 else \
            LayerTerms(0.0, _m.inf, t.agg_retention, t.agg_limit)
        layers.append(Layer(g.id, g.elts, terms))
    assert _fusable(layers, EngineConfig()) is not None
    fused, stats = run_aggregate_analysis_with_stats(layers, yet)
    assert stats.lookups == sum(len(l.elts) for l in layers) * int(yet.offsets[-1])
    for lay, y in zip(layers, fused):
        single = run_aggregate_analysis([lay], yet)[0].losses
        assert y.losses.tobytes() == single.tobytes()
        assert y.layer_id == lay.id
    small = yet.head(300)
    for lay in layers[:3]:
        want = _oracle_ylt(lay, small)
        got = run_aggregate_analysis(layers[:3], small)[layers.index(lay)].losses
        assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("n_layers", [2, 5, 7, 16])
def test_fused_layers_dense_overlap_and_odd_layer_counts(n_layers):
    """The fused kernel's fast path (events in <= 2 pool tables) and general
    path (3+) mixed in one sub-batch: a dense 10-table pool (most hot events
    sit in several tables), non-identity financial terms, layer counts that
    are not multiples of 4; each layer bitwise equal to its own K2 run and
    (first trials) to the reference loop."""
    rng = np.random.default_rng(7000 + n_layers)
    cat = 6_000
    pool = []
    for j in range(10):
        ids = np.sort(rng.choice(np.arange(1, cat + 1), size=int(rng.integers(900, 2_400)), replace=False))
        losses = rng.lognormal(0.0, 1.0, ids.shape[0]) * 1000.0
        losses[rng.random(ids.shape[0]) < 0.05] = 0.0  # explicit zero losses
        terms = FinancialTerms(float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.0, 300.0)),
                               float(rng.choice([math.inf, rng.uniform(500.0, 3000.0)])),
                               float(rng.uniform(0.1, 1.0)))
        pool.append(EventLossTable(cat, ids.astype(np.uint32), losses, terms))
    layers = []
    for i in range(n_layers):
        sel = np.sort(rng.choice(10, size=int(rng.integers(2, 9)), replace=False))
        occ_r, agg_r = float(rng.uniform(0, 800)), float(rng.uniform(0, 40_000))
        terms = LayerTerms(occ_r, float(rng.choice([math.inf, rng.uniform(1000, 5000)])), agg_r,
                           float(rng.choice([math.inf, rng.uniform(5_000, 60_000)])))
        layers.append(Layer(f"L{i}", tuple(pool[j] for j in sel), terms))
    yet = generate_yet(GeneratorSpec(seed=n_layers, catalog_size=cat, trial_count=1_500,
                                     events_per_trial_range=(1, 400),
                                     elt_size_range=(1, 10)), ids_only=True)
    fused = run_aggregate_analysis(layers, yet)
    for lay, y in zip(layers, fused):
        single = run_aggregate_analysis([lay], yet)[0].losses
        assert y.losses.tobytes() == single.tobytes(), lay.id
    small = yet.head(200)
    got = run_aggregate_analysis(layers, small)
    for lay, y in zip(layers, got):
        assert y.losses.tobytes() == _oracle_ylt(lay, small).tobytes(), lay.id
    # pre-combined variant (per-event occurrence table, K1-L): same bits
    from paper_1308_2066_b200.engine import layer_pool, simulate_layers_device
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    pool_elts, masks = layer_pool(layers)
    ptset = TableSet.from_elts(pool_elts, cat)
    dyet = DeviceYearEventTable(yet)
    terms = [lay.terms for lay in layers]
    exact = simulate_layers_device(dyet, ptset, masks, terms).cpu().numpy()
    for _ in range(2):  # second call reuses the cached table
        pre = simulate_layers_device(dyet, ptset, masks, terms, precombine=True).cpu().numpy()
        assert pre.tobytes() == exact.tobytes()
    assert all(exact[i].tobytes() == fused[i].losses.tobytes() for i in range(n_layers))
    via_entry = run_aggregate_analysis(layers, yet, EngineConfig(precombine=True))
    assert all(y.losses.tobytes() == fused[i].losses.tobytes() for i, y in enumerate(via_entry))


# ------------------------------------------------- the C ABI drop-in itself --

def test_c_abi_are_run_trials_matches_reference(instances):
    """are_run_trials: the reference run_trials argument list flattened to
    pointers (include/aggrisk_b200.h), as a cgo/ctypes binding would call it."""
    import ctypes

    lib = _native.load()
    for inst in instances[:200]:
        stacked = np.ascontiguousarray(inst.stacked)
        rows = np.arange(len(inst.layer.elts), dtype=np.int64)
        fin = [np.ascontiguousarray(a, dtype=np.float64) for a in inst.fin()]
        out = np.full(inst.yet.trial_count, -1.0)
        t = inst.layer.terms
        lookups = ctypes.c_int64()
        rc = lib.are_run_trials(inst.yet.event_ids.ctypes.data, inst.yet.event_ids.size,
                                inst.yet.offsets.ctypes.data, inst.yet.offsets.size,
                                stacked.ctypes.data, stacked.shape[0], stacked.shape[1],
                                rows.ctypes.data, rows.size, *(a.ctypes.data for a in fin),
                                t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit,
                                0, 0, inst.yet.trial_count, out.ctypes.data, 1, ctypes.byref(lookups))
        assert rc == 0, _native.last_error()
        assert out.tobytes() == inst.ylt.tobytes()
        assert lookups.value == rows.size * int(inst.yet.offsets[-1])
    # reference argument errors (_kernel.pyx:49-52) map to ARE_EINVAL
    inst = instances[0]
    stacked = np.ascontiguousarray(inst.stacked)
    rows = np.zeros(300, dtype=np.int64)
    ones = np.ones(300)
    rc = lib.are_run_trials(inst.yet.event_ids.ctypes.data, inst.yet.event_ids.size, inst.yet.offsets.ctypes.data,
                            inst.yet.offsets.size, stacked.ctypes.data, stacked.shape[0], stacked.shape[1],
                            rows.ctypes.data, 300, *(ones.ctypes.data for _ in range(4)), 0.0, 1.0, 0.0, 1.0,
                            0, 0, 1, np.empty(inst.yet.trial_count).ctypes.data, 1, None)
    assert rc == _native.ARE_EINVAL and "256" in _native.last_error()
    rc = lib.are_run_trials(inst.yet.event_ids.ctypes.data, inst.yet.event_ids.size, inst.yet.offsets.ctypes.data,
                            inst.yet.offsets.size, stacked.ctypes.data, stacked.shape[0], stacked.shape[1],
                            rows.ctypes.data, 1, *(ones.ctypes.data for _ in range(4)), 0.0, 1.0, 0.0, 1.0,
                            8, 0, 1, np.empty(inst.yet.trial_count).ctypes.data, 4, None)
    assert rc == _native.ARE_EINVAL and "scratch" in _native.last_error()
