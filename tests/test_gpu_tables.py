"""K1 direct-access tables built on the device, read back through the
reference's TableSet / DirectAccessTable API.

Mirrors the reference's table tests (pkg/tests/test_tables.py:22-128):
lookups of present / absent / out-of-range events, row stacking in ELT order,
selection order and errors, the build counter, and the dense memory account.
The rows are produced by k1_scatter_records on the GPU, so every read here
is a device -> host copy of what K2 later gathers from.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_1308_2066_b200.direct_access import (
    BYTES_PER_SLOT,
    TableSet,
    build_count,
    build_direct_table,
    lookup,
    memory_footprint,
)
from paper_1308_2066_b200.errors import EventOutOfRangeError
from paper_1308_2066_b200.portfolio import EventLossTable, FinancialTerms

pytestmark = pytest.mark.gpu


def _elt(records, catalog=10, terms=None):
    return EventLossTable.from_records(records, catalog_size=catalog, terms=terms)


def test_lookup_present_absent_and_explicit_zero():
    t = build_direct_table(_elt({4: 100.0, 9: 50.0, 6: 0.0}))
    assert (t.lookup(4), t.lookup(9), lookup(t, 4)) == (100.0, 50.0, 100.0)
    assert t.lookup(5) == 0.0 == t.lookup(6)  # absent and explicit zero read alike
    assert t.losses.shape == (11,) and t.losses[0] == 0.0  # slot 0 unused


@pytest.mark.parametrize("bad", [0, 11, -3])
def test_lookup_outside_catalog_raises(bad):
    with pytest.raises(EventOutOfRangeError):
        build_direct_table(_elt({4: 100.0})).lookup(bad)


def test_rows_are_read_only():
    t = build_direct_table(_elt({4: 100.0}))
    with pytest.raises(ValueError):
        t.losses[4] = 0.0


def test_rows_follow_elt_order_and_match_a_host_scatter():
    rng = np.random.default_rng(11)
    cat = 5_000
    elts = []
    for _ in range(6):
        ids = np.sort(rng.choice(np.arange(1, cat + 1), size=int(rng.integers(1, 900)), replace=False))
        elts.append(EventLossTable(cat, ids.astype(np.uint32), rng.lognormal(0.0, 1.0, ids.size) * 1e3))
    tset = TableSet.from_elts(elts)
    want = np.zeros((len(elts), cat + 1))
    for j, e in enumerate(elts):
        want[j, e.event_ids] = e.losses
    assert len(tset) == 6 and tset.stacked.shape == (6, cat + 1)
    assert tset.stacked.tobytes() == want.tobytes()
    assert tset.tables[3].losses.tobytes() == want[3].tobytes()
    assert [t.nonzero_count for t in tset.tables] == [int(np.count_nonzero(w)) for w in want]


def test_event_beyond_catalog_refused():
    with pytest.raises(EventOutOfRangeError):
        TableSet.from_elts([_elt({12: 1.0}, catalog=12)], catalog_size=10)


def test_from_tables_round_trip_and_mixed_catalogs():
    tables = [build_direct_table(_elt({i + 1: float(i + 1)})) for i in range(3)]
    tset = TableSet.from_tables(tables)
    assert tset.stacked[1].tobytes() == tables[1].losses.tobytes()
    with pytest.raises(ValueError):
        TableSet.from_tables([build_direct_table(_elt({1: 1.0}, catalog=5)),
                              build_direct_table(_elt({1: 1.0}, catalog=6))])


def test_selection_order_terms_and_errors():
    shares = (0.25, 0.5, 0.75)
    tset = TableSet.from_elts([_elt({1: 1.0}, terms=FinancialTerms(share=s)) for s in shares])
    rows, rate, _, _, share = tset.selection_arrays([2, 0])
    assert rows.tolist() == [2, 0] and share.tolist() == [0.75, 0.25] and rate.tolist() == [1.0, 1.0]
    assert tset.selection_arrays(None)[0].tolist() == [0, 1, 2]
    with pytest.raises(ValueError):
        tset.selection_arrays([])
    for bad in ([3], [-1]):
        with pytest.raises(IndexError):
            tset.selection_arrays(bad)


def test_build_counter_counts_builds_not_selections_or_plans():
    before = build_count()
    tset = TableSet.from_elts([_elt({1: 1.0}), _elt({2: 2.0})])
    assert build_count() == before + 1
    for _ in range(4):
        tset.plan(*tset.selection_arrays([0]))
        tset.selection_arrays(None)
    assert build_count() == before + 1


def test_memory_footprint_kats():
    fp = memory_footprint([build_direct_table(_elt({1: 1.0}, catalog=1000))])
    assert (fp.payload_slots, fp.total_bytes) == (1000, 8_008)
    tset = TableSet.from_elts([_elt({1: 1.0}, catalog=2_000_000) for _ in range(15)])
    fp = memory_footprint(tset.tables)
    assert (fp.table_count, fp.payload_slots, fp.payload_bytes) == (15, 30_000_000, 240_000_000)
    assert fp.overhead_bytes == 15 * BYTES_PER_SLOT
    small = TableSet.from_elts([_elt({1: 1.0}, catalog=50)] * 3)
    assert memory_footprint(small.tables).total_bytes == small.stacked.nbytes
