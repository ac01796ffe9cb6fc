"""Packed resident ids (are_yet_pack_device, csrc/k2_relay.cu).

A DeviceYearEventTable whose ids are validated and fit 21 bits keeps a second
copy of its ids packed three per 64-bit word; the relay kernel streams that
copy instead of the uint32 ids.  The YLT must stay bit-identical to the
reference run_trials (pkg/src/aggrisk/engine/_kernel.pyx:61-118) and to the
uint32 stream, for every trial length and alignment against the 96-id
blocks, and tables outside the layout's range must keep the uint32 path.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.portfolio import EventLossTable, FinancialTerms, LayerTerms, YearEventTable
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _packed_on(monkeypatch):
    monkeypatch.setenv("ARE_PACKED_IDS", "1")  # opt-in layout


CATALOG = 2_000_000


def _oracle(ids, offsets, stacked, fin, terms):
    out = np.empty(offsets.size - 1)
    oracle.run_trials_port(ids, offsets, stacked, np.arange(stacked.shape[0], dtype=np.int64),
                           *fin, terms.occ_retention, terms.occ_limit, terms.agg_retention, terms.agg_limit,
                           0, 0, offsets.size - 1, out)
    return out


@pytest.fixture(scope="module")
def tables():
    spec = GeneratorSpec(seed=91, catalog_size=CATALOG, trial_count=10, events_per_trial_range=(1, 2),
                         elt_count=5, elt_size_range=(150_000, 350_000))
    elts = []
    for i in range(spec.elt_count):
        e = generate_elt(spec, i)
        terms = FinancialTerms(exchange_rate=1.0 + 0.1 * i, event_retention=15.0 * i, event_limit=6_000.0 + 400 * i,
                               share=1.0 - 0.04 * i)
        elts.append(EventLossTable(e.catalog_size, e.event_ids, e.losses, terms))
    tset = TableSet.from_elts(elts)
    stacked = oracle.dense_tables(elts, CATALOG)
    fin = [np.array([getattr(e.terms, f) for e in elts], dtype=np.float64)
           for f in ("exchange_rate", "event_retention", "event_limit", "share")]
    return tset, stacked, fin


def _ragged(seed: int, n_trials: int):
    rng = np.random.default_rng(seed)
    # lengths around every 96-id block edge, empty and single-id trials, long
    # ones so the mean stays in the relay kernel's range
    pattern = [0, 1, 95, 96, 97, 191, 192, 193, 0, 287, 288, 289, 2, 1500, 0, 700, 3000, 383, 384, 385, 4096, 31]
    lengths = np.array([pattern[i % len(pattern)] for i in range(n_trials)], dtype=np.int64)
    rng.shuffle(lengths[: n_trials // 2])
    offsets = np.zeros(n_trials + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    ids = rng.integers(1, CATALOG + 1, size=int(offsets[-1]), dtype=np.uint32)
    return ids, offsets


def _simulate(dyet, tset, terms):
    plan = tset.plan(*tset.selection_arrays(None))
    return dyet.simulate_device(plan, terms).cpu().numpy(), plan


def test_packed_layout_words():
    """The packed words hold occurrences 96b + l + 32k in bits 21k..21k+20."""
    import torch
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    ids, offsets = _ragged(5, 701)
    dyet = DeviceYearEventTable(YearEventTable(CATALOG, ids, None, offsets))
    assert dyet.d_packed is not None
    words = dyet.d_packed.cpu().numpy().view(np.uint64)
    n = ids.size
    assert words.size == _native.load().are_packed_id_words(n) == (n + 95) // 96 * 32
    padded = np.zeros(words.size * 3, dtype=np.uint64)
    padded[:n] = ids
    blocks = padded.reshape(-1, 3, 32)  # [block][k][lane]
    want = blocks[:, 0, :] | (blocks[:, 1, :] << np.uint64(21)) | (blocks[:, 2, :] << np.uint64(42))
    assert np.array_equal(words, want.reshape(-1))
    torch.cuda.synchronize()


@pytest.mark.parametrize("seed", [1, 2])
def test_packed_relay_bitwise_equal_to_oracle_and_uint32(tables, seed, monkeypatch):
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    tset, stacked, fin = tables
    ids, offsets = _ragged(seed, 6_001)
    assert offsets[-1] / (offsets.size - 1) > 320  # the relay kernel's range
    host = YearEventTable(CATALOG, ids, None, offsets)
    packed = DeviceYearEventTable(host)
    monkeypatch.setenv("ARE_PACKED_IDS", "0")
    plain = DeviceYearEventTable(host)
    monkeypatch.setenv("ARE_PACKED_IDS", "1")
    assert packed.d_packed is not None and plain.d_packed is None
    for occ_ret, occ_lim in [(0.0, math.inf), (500.0, 10_000.0), (9_000.0, 1.0), (1e12, math.inf)]:
        terms = LayerTerms(occ_ret, occ_lim, 1_000.0, 2e6)
        got, plan = _simulate(packed, tset, terms)
        ref, _ = _simulate(plain, tset, terms)
        assert _native.plan_info(plan).relay_filter_bits > 0  # the relay kernel ran
        want = _oracle(ids, offsets, stacked, fin, terms)
        assert got.tobytes() == want.tobytes(), (occ_ret, occ_lim)
        assert ref.tobytes() == want.tobytes(), (occ_ret, occ_lim)


def test_packed_subrange_and_offset_first_trial(tables):
    """A launch over trials [first, last) starting mid-block."""
    import torch
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    tset, stacked, fin = tables
    ids, offsets = _ragged(7, 3_001)
    dyet = DeviceYearEventTable(YearEventTable(CATALOG, ids, None, offsets))
    terms = LayerTerms(500.0, 10_000.0, 1_000.0, 2e6)
    plan = tset.plan(*tset.selection_arrays(None))
    want = _oracle(ids, offsets, stacked, fin, terms)
    out = torch.full((offsets.size - 1,), -1.0, dtype=torch.float64, device=dyet.device)
    dyet.simulate_device(plan, terms, first=1_001, last=2_503, out=out)
    got = out.cpu().numpy()
    assert got[1_001:2_503].tobytes() == want[1_001:2_503].tobytes()
    assert (got[:1_001] == -1.0).all() and (got[2_503:] == -1.0).all()


def test_wide_ids_keep_the_uint32_stream():
    """A catalogue beyond 2^21 events builds no packed copy."""
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    cat = (1 << 21) + 10
    ids = np.array([1, cat, 5, (1 << 21)], dtype=np.uint32)
    offsets = np.array([0, 2, 4], dtype=np.int64)
    dyet = DeviceYearEventTable(YearEventTable(cat, ids, None, offsets))
    assert dyet.d_packed is None
