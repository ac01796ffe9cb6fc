"""A small relay-kernel run for compute-sanitizer (racecheck/synccheck/memcheck
take ~10 minutes on the parity suite's 2M-event catalog): 1,500 trials of
200-1,400 occurrences over a 100k catalog, checked against the oracle.
--packed: the same trials from a DeviceYearEventTable with the packed
resident ids (ARE_PACKED_IDS=1), so the relay kernel's packed stream runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import price_layer
from paper_1308_2066_b200.portfolio import LayerTerms
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet

spec = GeneratorSpec(seed=11, catalog_size=100_000, trial_count=1_500, events_per_trial_range=(200, 1400),
                     elt_count=6, elt_size_range=(3_000, 9_000))
yet = generate_yet(spec)
elts = [generate_elt(spec, i) for i in range(spec.elt_count)]
tset = TableSet.from_elts(elts, spec.catalog_size)
stacked = oracle.dense_tables(elts, spec.catalog_size)
fin = [np.array([getattr(e.terms, f) for e in elts]) for f in ("exchange_rate", "event_retention", "event_limit", "share")]
packed = "--packed" in sys.argv
if packed:
    os.environ["ARE_PACKED_IDS"] = "1"
    from paper_1308_2066_b200.resident import DeviceYearEventTable
    dyet = DeviceYearEventTable(yet)
    assert dyet.d_packed is not None
for occ in [(500.0, 10_000.0), (0.0, float("inf"))]:
    terms = LayerTerms(*occ, 2_000.0, 1e6)
    if packed:
        got = dyet.simulate_device(tset.plan(*tset.selection_arrays(None)), terms).cpu().numpy()
    else:
        got, _ = price_layer(yet, tset, None, terms)
    want = np.zeros(yet.trial_count)
    oracle.run_trials_port(yet.event_ids, yet.offsets, stacked, np.arange(len(elts), dtype=np.int64), *fin,
                           *occ, 2_000.0, 1e6, 0, 0, yet.trial_count, want)
    assert got.tobytes() == want.tobytes(), occ
info = _native.plan_info(tset.plan(*tset.selection_arrays(None)))
assert info.relay, "the relay kernel did not run"
print("relay small run ok" + (" (packed ids)" if packed else ""))
