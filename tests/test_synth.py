"""The generator restatement reproduces the reference generator byte for byte
(digests recorded from /root/reference by tests/golden/make_golden.py)."""

from __future__ import annotations

import hashlib

import numpy as np

from paper_1308_2066_b200.synth import GeneratorSpec, bulk_yet, generate_elt, generate_layer, generate_yet


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_seed31_yet_and_elts_match_reference(golden):
    g = golden["seed31"]
    spec = GeneratorSpec(seed=31, catalog_size=2_000, trial_count=10_000,
                         events_per_trial_range=(10, 50), elt_count=3, elt_size_range=(200, 800))
    yet = generate_yet(spec)
    assert sha(yet.event_ids) == g["yet_ids_sha256"]
    assert sha(yet.offsets) == g["yet_offsets_sha256"]
    assert sha(yet.timestamps) == g["yet_timestamps_sha256"]
    assert [sha(e.event_ids, e.losses) for e in (generate_elt(spec, i) for i in range(3))] == g["elt_sha256"]
    ids_only = generate_yet(spec, ids_only=True)
    assert ids_only.timestamps is None
    assert ids_only.event_ids.tobytes() == yet.event_ids.tobytes()


def test_c1_inputs_match_reference(golden):
    c1 = golden["c1"]
    spec = GeneratorSpec(seed=2066, catalog_size=2_000_000, trial_count=10_000,
                         events_per_trial_range=(1000, 1000), elt_count=15,
                         elt_size_range=(10_000, 30_000), loss_scale=1000.0)
    yet = generate_yet(spec, ids_only=True)
    assert sha(yet.event_ids) == c1["yet_ids_sha256"]
    assert sha(yet.offsets) == c1["yet_offsets_sha256"]
    elts = [generate_elt(spec, i) for i in range(15)]
    assert [sha(e.event_ids, e.losses) for e in elts] == c1["elt_sha256"]
    layer = generate_layer(spec, 0, elts)
    t = layer.terms
    assert [t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit] == c1["generated_layer_terms"]
    assert [elts.index(e) for e in layer.elts] == c1["layer_elt_indices"]


def test_bulk_yet_is_partition_invariant():
    whole = bulk_yet(5, 2_000_000, 0, 10_000, 100, threads=4, block=1024)
    a = bulk_yet(5, 2_000_000, 0, 3_333, 100, threads=2, block=1024)
    b = bulk_yet(5, 2_000_000, 3_333, 10_000, 100, threads=3, block=1024)
    assert np.concatenate([a.event_ids, b.event_ids]).tobytes() == whole.event_ids.tobytes()
    assert whole.event_ids.min() >= 1 and whole.event_ids.max() <= 2_000_000
    assert whole.offsets[-1] == 1_000_000
