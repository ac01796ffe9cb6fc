"""Writes the golden fixtures under tests/golden/ from the REFERENCE package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference `aggrisk` package from /root/reference/pkg/src and
its test oracle from /root/reference/pkg/tests, runs them, and stores inputs
plus outputs as small .npz/.json fixtures.  Nothing at test time reads
/root/reference; the tests compare our oracle port and the CUDA path against
these files.  The reference engine runs with backend="python"
(engine/_fallback.py), which the reference's own suite pins bit-identical to
the compiled Cython kernel (pkg/tests/test_engine.py:105-117); the script
also cross-checks against the Cython kernel compiled into oracle/_ref.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path[:0] = [REF_SRC, REF_TESTS]

import oracle as ref_oracle  # noqa: E402  (reference pkg/tests/oracle.py)
from aggrisk import engine as ref_engine  # noqa: E402
from aggrisk import metrics as ref_metrics  # noqa: E402
from aggrisk.generate import GeneratorSpec, generate_elt, generate_layer, generate_yet  # noqa: E402
from aggrisk.model import EventLossTable, Layer, LayerTerms, Trial, YearEventTable  # noqa: E402
from aggrisk.tables import TableSet  # noqa: E402

PY = ref_engine.EngineConfig(backend="python")


def _cython_kernel():
    path = os.path.join(REPO, "oracle", "_ref")
    for f in os.listdir(path) if os.path.isdir(path) else []:
        if f.startswith("_kernel") and f.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_kernel", os.path.join(path, f))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _pack_instances(instances):
    """Flatten (layer, yet, ylt) triples into concatenated arrays."""
    cat, lterms, n_elts, yet_off, trial_off, ids = [], [], [], [0], [], []
    elt_off, elt_ids, elt_loss, fin = [0], [], [], []
    ylt_ref, ylt_oracle, ylt_off = [], [], [0]
    occ_base = 0
    for layer, yet, ylt, ylt_o in instances:
        cat.append(yet.catalog_size)
        t = layer.terms
        lterms.append([t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit])
        n_elts.append(len(layer.elts))
        for e in layer.elts:
            elt_ids.append(e.event_ids)
            elt_loss.append(e.losses)
            elt_off.append(elt_off[-1] + e.record_count)
            ft = e.terms
            fin.append([ft.exchange_rate, ft.event_retention, ft.event_limit, ft.share])
        trial_off.append(yet.offsets + occ_base)
        occ_base += int(yet.offsets[-1])
        yet_off.append(yet_off[-1] + yet.trial_count)
        ids.append(yet.event_ids)
        ylt_ref.append(ylt)
        ylt_oracle.append(ylt_o)
        ylt_off.append(ylt_off[-1] + len(ylt))
    return dict(
        catalog=np.array(cat, np.int64),
        layer_terms=np.array(lterms, np.float64),
        n_elts=np.array(n_elts, np.int64),
        elt_offsets=np.array(elt_off, np.int64),
        elt_ids=np.concatenate(elt_ids).astype(np.uint32),
        elt_losses=np.concatenate(elt_loss).astype(np.float64),
        fin_terms=np.array(fin, np.float64),
        # per instance: trial_offsets slice [yet_off[i], yet_off[i+1]+i] ...
        trial_bounds=np.array(yet_off, np.int64),
        trial_offsets=np.concatenate(
            [o if i == 0 else o[1:] for i, o in enumerate(trial_off)]
        ).astype(np.int64),
        event_ids=np.concatenate(ids).astype(np.uint32),
        ylt=np.concatenate(ylt_ref).astype(np.float64),
        ylt_naive_oracle=np.concatenate(ylt_oracle).astype(np.float64),
        ylt_bounds=np.array(ylt_off, np.int64),
    )


def random_instances(seed: int, count: int):
    """pkg/tests/test_acceptance.py:47-63 -- 1000 instances, rng 1001."""
    rng = np.random.default_rng(seed)
    out = []
    ker = _cython_kernel()
    for _ in range(count):
        layer, yet = ref_oracle.random_instance(rng, max_trials=100, max_events=100, max_elts=5)
        ylt = ref_engine.run_aggregate_analysis([layer], yet, PY)[0].losses
        if ker is not None:  # compiled reference must agree bitwise
            tset = TableSet.from_elts(layer.elts, yet.catalog_size)
            sel, r, re, li, sh = tset.selection_arrays(None)
            o = np.empty(yet.trial_count)
            t = layer.terms
            ker.run_trials(yet.event_ids, yet.offsets, tset.stacked, sel, r, re, li, sh,
                           t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit,
                           0, 0, yet.trial_count, o, np.empty(1))
            assert o.tobytes() == ylt.tobytes()
        naive = np.asarray(ref_oracle.layer_ylt(layer, yet), dtype=np.float64)
        out.append((layer, yet, ylt, naive))
    return out


def kats() -> dict:
    """Known answers from the reference suite, recomputed by the reference."""
    elt = EventLossTable.from_records({4: 100.0, 9: 50.0}, catalog_size=10)
    layer = Layer("L", (elt,), LayerTerms(10.0, 60.0, 0.0, 150.0))
    worked = ref_engine.analyse_trial(Trial.from_events([4, 9, 4]), layer, cfg=PY)
    one = EventLossTable.from_records({1: 10.0}, catalog_size=5)
    multi = ref_engine.run_aggregate_analysis(
        [Layer("first", (one,), LayerTerms()), Layer("second", (one,), LayerTerms(occ_limit=4.0))],
        YearEventTable.from_trials([Trial.from_events([1])], catalog_size=5), PY)
    ramp = np.arange(1, 1001, dtype=np.float64)
    ramp10 = np.arange(1, 11, dtype=np.float64)
    return {
        "worked_example": worked,                                    # test_engine.py:27-38
        "multi_layer": [float(y.losses[0]) for y in multi],          # test_engine.py:137-147
        "fin_terms_30_2_10_40_half": ref_engine.apply_financial_terms(
            30.0, ref_engine.FinancialTerms(2.0, 10.0, 40.0, 0.5)),  # test_terms.py:23-26
        "pml_ramp1000_rp100": ref_metrics.pml(ramp, 100.0),          # test_metrics.py:16-18
        "tvar_ramp1000_rp100": ref_metrics.tvar(ramp, 100.0),
        "ep_ramp1000": [list(p) for p in ref_metrics.ep_curve(ramp, [2.0, 10.0, 100.0]).points],
        "pml_ramp10_rp10": ref_metrics.pml(ramp10, 10.0),
        "tvar_ramp10_rp10": ref_metrics.tvar(ramp10, 10.0),
        "pml_10_110_rp3": ref_metrics.pml(np.arange(10.0, 110.0, 10.0), 3.0),
    }


def split_cases() -> list:
    """engine/__init__.py:151-159 on random offsets -- the trial->GPU partition."""
    rng = np.random.default_rng(4242)
    cases = []
    for _ in range(300):
        n = int(rng.integers(1, 400))
        lens = rng.integers(0, 50, size=n)
        if rng.random() < 0.2:
            lens[:] = int(rng.integers(1, 20))
        offsets = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=offsets[1:])
        parts = int(rng.integers(1, 40))
        got = ref_engine._split_by_events(offsets, parts)
        cases.append({"lens": lens.tolist(), "parts": parts, "batches": [list(b) for b in got]})
    return cases


def metric_cases():
    """metrics.py:29-115 on random YLTs (cf. test_acceptance.py:257-283)."""
    rng = np.random.default_rng(1004)
    ylts, bounds, rps_all, pmls, tvars = [], [0], [], [], []
    for _ in range(300):
        n = int(rng.integers(2, 400))
        losses = rng.lognormal(0.0, 1.5, n) * 100.0
        if rng.random() < 0.1:
            losses[rng.random(n) < 0.5] = 0.0
        if rng.random() < 0.1:
            losses = np.round(losses / 50.0) * 50.0  # ties
        rps = sorted(float(rng.uniform(1.0 + 1e-9, n)) for _ in range(4))
        ylts.append(losses)
        bounds.append(bounds[-1] + n)
        rps_all.append(rps)
        pmls.append([ref_metrics.pml(losses, rp) for rp in rps])
        tvars.append([ref_metrics.tvar(losses, rp) for rp in rps])
    return dict(losses=np.concatenate(ylts), bounds=np.array(bounds, np.int64),
                rps=np.array(rps_all), pml=np.array(pmls), tvar=np.array(tvars))


def seed31_digest() -> dict:
    """test_acceptance.py:93-118 -- generator + engine digest 5ebdd83b8ee0."""
    spec = GeneratorSpec(seed=31, catalog_size=2_000, trial_count=10_000,
                         events_per_trial_range=(10, 50), elt_count=3, elt_size_range=(200, 800))
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(spec.elt_count)]
    layer = Layer("det", tuple(elts), LayerTerms(500.0, 20_000.0, 0.0, 300_000.0))
    ylt = ref_engine.run_aggregate_analysis([layer], yet, PY)[0].losses
    return {
        "yet_ids_sha256": sha(yet.event_ids),
        "yet_offsets_sha256": sha(yet.offsets),
        "yet_timestamps_sha256": sha(yet.timestamps),
        "elt_sha256": [sha(e.event_ids, e.losses) for e in elts],
        "ylt_sha256": sha(ylt),
    }


def c1_fixture():
    """seed 2066, catalog 2M, 10k x 1000, 15 ELTs, Cat XL+Agg XL.

    Inputs are regenerated at test time by our generator port (digests pin
    them); the fixture keeps the reference YLT and its PML/TVaR.
    """
    spec = GeneratorSpec(seed=2066, catalog_size=2_000_000, trial_count=10_000,
                         events_per_trial_range=(1000, 1000), elt_count=15,
                         elt_size_range=(10_000, 30_000), loss_scale=1000.0, layer_count=1)
    yet = generate_yet(spec)
    elts = [generate_elt(spec, i) for i in range(spec.elt_count)]
    gen_layer = generate_layer(spec, 0, elts)
    terms = LayerTerms(500.0, 10_000.0, 140_000.0, 66_000.0)
    layer = Layer(gen_layer.id, gen_layer.elts, terms)
    ker = _cython_kernel()
    tset = TableSet.from_elts(layer.elts, yet.catalog_size)
    sel, r, re, li, sh = tset.selection_arrays(None)
    ylt = np.empty(yet.trial_count)
    ker.run_trials(yet.event_ids, yet.offsets, tset.stacked, sel, r, re, li, sh,
                   terms.occ_retention, terms.occ_limit, terms.agg_retention, terms.agg_limit,
                   0, 0, yet.trial_count, ylt, np.empty(1))
    rps = [2.0, 10.0, 50.0, 100.0, 250.0, 1000.0]
    meta = {
        "yet_ids_sha256": sha(yet.event_ids),
        "yet_offsets_sha256": sha(yet.offsets),
        "layer_elt_indices": [elts.index(e) for e in layer.elts],
        "elt_sha256": [sha(e.event_ids, e.losses) for e in elts],
        "generated_layer_terms": [gen_layer.terms.occ_retention, gen_layer.terms.occ_limit,
                                  gen_layer.terms.agg_retention, gen_layer.terms.agg_limit],
        "rps": rps,
        "pml": [ref_metrics.pml(ylt, rp) for rp in rps],
        "tvar": [ref_metrics.tvar(ylt, rp) for rp in rps],
        "ylt_sha256": sha(ylt),
    }
    return meta, ylt


def are1_fixture() -> dict:
    """A small ARE1 binary YET written by the reference (io.py:150-175)."""
    from aggrisk.io import save_yet

    spec = GeneratorSpec(seed=5, catalog_size=3_000, trial_count=400,
                         events_per_trial_range=(0, 60), elt_count=1, elt_size_range=(10, 20))
    yet = generate_yet(spec)
    path = os.path.join(HERE, "yet_small.are1")
    save_yet(yet, path, format="binary")
    return {"ids_sha256": sha(yet.event_ids), "offsets_sha256": sha(yet.offsets),
            "timestamps_sha256": sha(yet.timestamps), "catalog": yet.catalog_size,
            "trials": yet.trial_count}


def main() -> None:
    out = {}
    out["are1"] = are1_fixture()
    out["kats"] = kats()
    out["split_by_events"] = split_cases()
    out["seed31"] = seed31_digest()
    assert out["seed31"]["ylt_sha256"].startswith("5ebdd83b8ee0"), out["seed31"]
    c1_meta, c1_ylt = c1_fixture()
    out["c1"] = c1_meta
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.save(os.path.join(HERE, "c1_ylt.npy"), c1_ylt)
    np.savez_compressed(os.path.join(HERE, "random_instances_1001.npz"),
                        **_pack_instances(random_instances(1001, 1000)))
    np.savez_compressed(os.path.join(HERE, "metrics_1004.npz"), **metric_cases())
    print("wrote golden fixtures to", HERE)


if __name__ == "__main__":
    main()
