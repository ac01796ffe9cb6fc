"""Bounds-checked run of the relay kernel's uint32 and packed streams
(compute-sanitizer is closed on the GPU pool).  Build the checked library
first:

    make -C paper_1308_2066_b200/csrc OUT=$PWD/build/lib_bounds.so EXTRA=-DARE_KR_BOUNDS=1
    ARE_LIB=build/lib_bounds.so python scripts/packed_bounds.py

Ragged trials around every 96/192-id block edge, launches over sub-ranges
starting mid-block, the last trial ending at the array's end; every YLT is
compared with the oracle and the plan's error word must stay 0 (bit 2: a
packed word read outside the array, bit 4: a queue holding more than its
capacity)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ARE_PACKED_IDS"] = "1"
import numpy as np
import torch

import oracle
from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.portfolio import LayerTerms, YearEventTable
from paper_1308_2066_b200.resident import DeviceYearEventTable
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt

CAT = 200_000
spec = GeneratorSpec(seed=5, catalog_size=CAT, trial_count=10, events_per_trial_range=(1, 2), elt_count=5,
                     elt_size_range=(10_000, 30_000))
elts = [generate_elt(spec, i) for i in range(spec.elt_count)]
tset = TableSet.from_elts(elts, CAT)
stacked = oracle.dense_tables(elts, CAT)
fin = [np.array([getattr(e.terms, f) for e in elts]) for f in ("exchange_rate", "event_retention", "event_limit", "share")]
lib = _native.load()
checked = 0
for seed in range(6):
    rng = np.random.default_rng(seed)
    pattern = [0, 1, 95, 96, 97, 191, 192, 193, 287, 288, 289, 383, 384, 385, 31, 500, 1500, 4000]
    lengths = rng.choice(pattern, size=2_001 + seed)
    lengths[-1] = 97 + seed  # the last trial ends inside the final block
    offsets = np.zeros(lengths.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    ids = rng.integers(1, CAT + 1, size=int(offsets[-1]), dtype=np.uint32)
    for packed in ("1", "0"):
        os.environ["ARE_PACKED_IDS"] = packed
        dyet = DeviceYearEventTable(YearEventTable(CAT, ids, None, offsets))
        assert (dyet.d_packed is not None) == (packed == "1")
        for occ in [(500.0, 10_000.0), (0.0, float("inf"))]:
            terms = LayerTerms(*occ, 2_000.0, 1e6)
            plan = tset.plan(*tset.selection_arrays(None))
            want = np.zeros(lengths.size)
            oracle.run_trials_port(ids, offsets, stacked, np.arange(len(elts), dtype=np.int64), *fin, *occ,
                                   2_000.0, 1e6, 0, 0, lengths.size, want)
            for first, last in [(0, lengths.size), (seed * 37 + 1, lengths.size), (3, lengths.size // 2)]:
                out = torch.zeros(lengths.size, dtype=torch.float64, device=dyet.device)
                dyet.simulate_device(plan, terms, first=first, last=last, out=out)
                torch.cuda.synchronize()
                rc = lib.are_check_errors(plan.value, None)
                assert rc == 0, (seed, packed, first, last, _native.last_error() if hasattr(_native, "last_error") else rc)
                got = out.cpu().numpy()
                assert got[first:last].tobytes() == want[first:last].tobytes(), (seed, packed, first, last)
                checked += 1
assert _native.plan_info(tset.plan(*tset.selection_arrays(None))).relay, "the relay kernel did not run"
print(f"bounds-checked relay runs ok: {checked} launches (packed and uint32), error word 0, YLT = oracle")
