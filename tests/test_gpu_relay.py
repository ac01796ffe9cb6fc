"""The relay kernel (csrc/k2_relay.cu) against the reference kernel.

k2_relay skips every event whose occurrence value is +-0 under the launch's
occurrence terms (the per-terms "contributing" filter, k1_relay_filter) and
folds on a separate warp; the YLT must still be bit-identical to the
reference run_trials (pkg/src/aggrisk/engine/_kernel.pyx:61-118).  These
cases move the occurrence retention across the loss distribution (from
"every hot event contributes" to "almost none does"), reuse one plan for
more distinct terms than the per-plan filter cache holds (eviction path), and
mix multi-table events (records with inline 2nd/3rd entries and overflow
beyond).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import price_layer
from paper_1308_2066_b200.portfolio import EventLossTable, FinancialTerms, LayerTerms
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet

pytestmark = pytest.mark.gpu


def _oracle(yet, stacked, fin, terms):
    out = np.empty(yet.trial_count)
    oracle.run_trials_port(yet.event_ids, yet.offsets, stacked, np.arange(stacked.shape[0], dtype=np.int64),
                           *fin, terms.occ_retention, terms.occ_limit, terms.agg_retention, terms.agg_limit,
                           0, 0, yet.trial_count, out)
    return out


@pytest.fixture(scope="module")
def case():
    # long trials (the relay kernel runs above 145 occurrences per trial) over
    # a catalog larger than the shared-memory filter, 6 ELTs with overlap so
    # some events sit in 4+ tables (overflow entries beyond the record)
    spec = GeneratorSpec(seed=77, catalog_size=2_000_000, trial_count=3_000, events_per_trial_range=(400, 1500),
                         elt_count=6, elt_size_range=(150_000, 400_000))
    yet = generate_yet(spec)
    elts = []
    for i in range(spec.elt_count):
        e = generate_elt(spec, i)
        terms = FinancialTerms(exchange_rate=1.0 + 0.1 * i, event_retention=20.0 * i, event_limit=5_000.0 + 500 * i,
                               share=1.0 - 0.05 * i)
        elts.append(EventLossTable(e.catalog_size, e.event_ids, e.losses, terms))
    tset = TableSet.from_elts(elts)
    stacked = oracle.dense_tables(elts, spec.catalog_size)
    fin = [np.array([getattr(e.terms, f) for e in elts], dtype=np.float64)
           for f in ("exchange_rate", "event_retention", "event_limit", "share")]
    counts = (stacked[:, 1:] != 0).sum(axis=0)
    assert counts.max() >= 4, "the case must include events in 4+ tables"
    return yet, elts, tset, stacked, fin


OCC_TERMS = [(0.0, math.inf), (500.0, 10_000.0), (2_000.0, 3_000.0), (4_000.0, math.inf), (9_000.0, 1.0),
             (0.0, 250.0), (1e12, math.inf)]


def test_occurrence_terms_sweep_and_filter_eviction(case):
    yet, elts, tset, stacked, fin = case
    for rounds in range(2):  # the second round re-meets evicted and cached filters
        for occ_ret, occ_lim in OCC_TERMS:
            terms = LayerTerms(occ_ret, occ_lim, 1_000.0, 2e6)
            got, lookups = price_layer(yet, tset, None, terms)
            want = _oracle(yet, stacked, fin, terms)
            assert got.tobytes() == want.tobytes(), (rounds, occ_ret, occ_lim)
            assert lookups == len(elts) * yet.event_ids.size


def test_kernel_paths_agree_bitwise(case):
    """AUTO (the relay kernel here) against the dense literal loop, which
    performs every lookup: both bit-identical to the reference."""
    yet, elts, tset, stacked, fin = case
    from paper_1308_2066_b200.engine import EngineConfig

    terms = LayerTerms(700.0, 8_000.0, 5_000.0, 1e5)
    hot, _ = price_layer(yet, tset, None, terms)
    dense, _ = price_layer(yet, tset, None, terms, EngineConfig(variant="dense"))
    assert hot.tobytes() == dense.tobytes() == _oracle(yet, stacked, fin, terms).tobytes()


def test_ragged_trials_across_the_stream(case):
    """The relay warps stream their trials back to back (a trial's first ids
    are loaded while the previous trial is still filtered; a trial's final
    batch is published with the next push).  Mix empty trials, single-id
    trials, trials of exactly 31/32/33/128/129 ids and long ones (mean length
    stays above the short-trial kernel's range), under terms where every,
    some and no hot event contributes."""
    yet, elts, tset, stacked, fin = case
    from paper_1308_2066_b200.portfolio import YearEventTable

    rng = np.random.default_rng(2066)
    pattern = [0, 1, 0, 0, 31, 32, 33, 128, 129, 1500, 0, 2, 700, 3000, 0, 5, 257, 1, 0, 4096]
    lengths = np.array([pattern[i % len(pattern)] for i in range(9_001)], dtype=np.int64)
    rng.shuffle(lengths[: len(lengths) // 2])
    offsets = np.zeros(lengths.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    assert offsets[-1] / lengths.size > 145  # the relay kernel's range
    src = yet.event_ids
    ids = src[rng.integers(0, src.size, size=int(offsets[-1]))]
    ragged = YearEventTable(yet.catalog_size, ids, None, offsets)
    for occ_ret, occ_lim in [(0.0, math.inf), (500.0, 10_000.0), (9_000.0, 1.0), (1e12, math.inf)]:
        terms = LayerTerms(occ_ret, occ_lim, 1_000.0, 2e6)
        got, lookups = price_layer(ragged, tset, None, terms)
        want = _oracle(ragged, stacked, fin, terms)
        assert got.tobytes() == want.tobytes(), (occ_ret, occ_lim)
        assert lookups == len(elts) * ids.size


def test_short_trials_in_the_relay_range(case):
    """Mean trial lengths just above the k2_pair crossover (145-250
    occurrences) run the relay kernel: many trials per warp, most final
    batches partial, some trials with no contributing event at all."""
    yet, elts, tset, stacked, fin = case
    from paper_1308_2066_b200.portfolio import YearEventTable

    rng = np.random.default_rng(1308)
    for lo, hi in [(100, 200), (150, 350)]:
        lengths = rng.integers(lo, hi, size=12_001)
        offsets = np.zeros(lengths.size + 1, dtype=np.int64)
        np.cumsum(lengths, out=offsets[1:])
        assert 145 < offsets[-1] / lengths.size <= 320
        ids = yet.event_ids[rng.integers(0, yet.event_ids.size, size=int(offsets[-1]))]
        short = YearEventTable(yet.catalog_size, ids, None, offsets)
        for occ_ret, occ_lim in [(500.0, 10_000.0), (9_000.0, 1.0)]:
            terms = LayerTerms(occ_ret, occ_lim, 1_000.0, 2e6)
            got, _ = price_layer(short, tset, None, terms)
            assert got.tobytes() == _oracle(short, stacked, fin, terms).tobytes(), (lo, hi, occ_ret)


def test_nan_inf_and_multi_entry_records():
    """The 16-byte relay record: one or two entries inline, 3+ entries or a
    NaN among the first two through the NaN-tagged overflow form.  NaN and
    +inf losses, zero losses and events in 1-4 tables, long trials (the relay
    range); NaNs must sit in the same trials, every other value bitwise."""
    from paper_1308_2066_b200.portfolio import YearEventTable

    rng = np.random.default_rng(4)
    cat = 5_000
    elts = []
    for j in range(4):
        ids = np.sort(rng.choice(np.arange(1, cat + 1), 2_500, replace=False)).astype(np.uint32)
        losses = rng.lognormal(0, 1, ids.size) * 300.0
        losses[rng.choice(ids.size, 3, replace=False)] = np.nan  # few enough that most trials miss them
        losses[rng.choice(ids.size, 3, replace=False)] = np.inf
        losses[rng.random(ids.size) < 0.05] = 0.0
        elts.append(EventLossTable(cat, ids, losses, FinancialTerms(1.0 + 0.25 * j, 10.0 * j, 4_000.0 if j % 2 else math.inf,
                                                                     1.0 - 0.1 * j)))
    tset = TableSet.from_elts(elts, cat)
    stacked = oracle.dense_tables(elts, cat)
    fin = [np.array([getattr(e.terms, f) for e in elts], dtype=np.float64)
           for f in ("exchange_rate", "event_retention", "event_limit", "share")]
    counts = (stacked[:, 1:] != 0).sum(axis=0)
    assert counts.max() == 4 and (counts == 2).any() and (counts == 3).any()
    lengths = rng.integers(300, 600, size=400)
    offsets = np.zeros(lengths.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    yet = YearEventTable(cat, rng.integers(1, cat + 1, int(offsets[-1])).astype(np.uint32), None, offsets)
    from paper_1308_2066_b200.engine import EngineConfig

    for occ_ret, occ_lim in [(0.0, math.inf), (200.0, 5_000.0)]:
        terms = LayerTerms(occ_ret, occ_lim, 1_000.0, math.inf)
        want = _oracle(yet, stacked, fin, terms)
        assert np.isnan(want).any() and not np.isnan(want).all()
        # exact records, and pre-combined ones ({comb, +0.0}; a NaN comb tagged)
        for cfg in (EngineConfig(), EngineConfig(precombine=True)):
            got, _ = price_layer(yet, tset, None, terms, cfg)
            assert np.array_equal(np.isnan(got), np.isnan(want)), cfg
            ok = ~np.isnan(want)
            assert got[ok].tobytes() == want[ok].tobytes(), (occ_ret, occ_lim, cfg)


def test_out_of_range_id_in_a_long_trial_raises(case):
    """The relay kernel's per-id range check (unvalidated host YETs): an id
    beyond the catalog inside a long trial raises EventOutOfRangeError, as
    the reference's analyse_trial / validation would."""
    yet, elts, tset, stacked, fin = case
    from paper_1308_2066_b200.errors import EventOutOfRangeError
    from paper_1308_2066_b200.portfolio import YearEventTable

    ids = np.array(yet.event_ids[: 600 * 50], dtype=np.uint32)
    ids[12_345] = yet.catalog_size + 7
    bad = YearEventTable(yet.catalog_size, ids, None, np.arange(51, dtype=np.int64) * 600)
    with pytest.raises(EventOutOfRangeError):
        price_layer(bad, tset, None, LayerTerms(500.0, 10_000.0, 1_000.0, 2e6))
