"""The plug-in seam under the reference's own threaded driver.

The reference calls the backend's run_trials concurrently from a
ThreadPoolExecutor over disjoint trial ranges (engine/__init__.py:193-200)
and its service shares one pool across requests (service.py:117-123).  Here
8 workers drive engine.run_trials with 12 distinct (selection, financial
terms) plans over one read-only `stacked` array -- more plans than the
device cache keeps, so evictions happen while other threads launch -- and
every range must be bitwise equal to the oracle."""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_1308_2066_b200 import engine
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet

pytestmark = pytest.mark.gpu


def test_concurrent_run_trials_with_plan_evictions():
    spec = GeneratorSpec(seed=99, catalog_size=5000, trial_count=2000, events_per_trial_range=(20, 180),
                         elt_count=15, elt_size_range=(300, 1500))
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(15)]
    stacked = oracle.dense_tables(elts, spec.catalog_size)
    stacked.setflags(write=False)  # read-only: the device copy is cached (reference tables.py:84)
    rng = np.random.default_rng(4)
    combos = []
    for k in range(12):
        rows = rng.choice(15, size=int(rng.integers(2, 9)), replace=False).astype(np.int64)
        n = rows.size
        fin = [rng.uniform(0.5, 2.0, n), rng.uniform(0, 50, n), rng.uniform(200, 5000, n), rng.uniform(0.2, 1, n)]
        terms = (float(rng.uniform(0, 100)), float(rng.uniform(500, 5000)), float(rng.uniform(0, 2000)),
                 float(rng.uniform(5000, 40000)))
        combos.append((rows, [np.ascontiguousarray(a) for a in fin], terms))
    ids, offs = yet.event_ids, yet.offsets
    batches = oracle.split_by_events(offs, 8)
    outs = [np.zeros(yet.trial_count) for _ in combos]

    def task(job):
        c, (t0, t1) = job
        rows, fin, terms = combos[c]
        return engine.run_trials(ids, offs, stacked, rows, *fin, *terms, 0, t0, t1, outs[c])

    jobs = [(c, b) for _ in range(2) for c in range(len(combos)) for b in batches]
    rng.shuffle(jobs)
    with ThreadPoolExecutor(max_workers=8) as ex:
        counts = list(ex.map(task, jobs))
    kind = "reference" if oracle.ref_kernel() is not None else "port"
    for c, (rows, fin, terms) in enumerate(combos):
        want, _ = oracle.run_layer_cpu(ids, offs, np.ascontiguousarray(stacked[rows]), fin, terms, kernel=kind)
        assert outs[c].tobytes() == want.tobytes(), f"combination {c}"
    assert sum(counts) == 2 * sum(combos[c][0].size for c in range(len(combos))) * int(offs[-1])


def test_calls_on_another_device_restore_the_current_device():
    """use_device() inside the library must not leak into the caller's thread
    (a plan on GPU 1 used while torch's current device is 0)."""
    import torch

    n = torch.cuda.device_count()
    torch.cuda.set_device(n - 1)
    spec = GeneratorSpec(seed=1, catalog_size=1000, trial_count=50, events_per_trial_range=(1, 30),
                         elt_count=2, elt_size_range=(50, 100))
    yet = generate_yet(spec)
    stacked = oracle.dense_tables([generate_elt(spec, i) for i in range(2)], 1000)
    out = np.zeros(50)
    torch.cuda.set_device(0)
    engine.run_trials(yet.event_ids, yet.offsets, stacked, np.arange(2, dtype=np.int64), np.ones(2), np.zeros(2),
                      np.full(2, np.inf), np.ones(2), 0.0, np.inf, 0.0, np.inf, 0, 0, 50, out)
    assert torch.cuda.current_device() == 0
