"""Writes tests/golden/validation.json.gz from the REFERENCE `validate_portfolio`.

Run in the build container (where /root/reference exists):

    python tests/golden/make_validation.py

Every case is built with the reference's own model types
(pkg/src/aggrisk/model.py), validated by the reference's
`validate_portfolio` (model.py:360-404), and stored as raw arrays (YET ids,
timestamps, offsets; each ELT's ids, losses and financial terms; each
layer's terms) together with the reference report as its `str(v)` list
("[category] message", model.py:306-313).  The cases cover the reference's
own per-category tests (pkg/tests/test_model.py:138-258), this repo's
host/K0 cases, NaN timestamps, id 0, over-long and empty trials, boundary
drops, combined violations, and a seeded random mix.  The tests rebuild each
case from the arrays with this repo's types and require byte-equal lists
from the host path and from the K0 device path.
"""

from __future__ import annotations

import gzip
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from aggrisk.model import (  # noqa: E402
    MAX_TRIAL_LENGTH,
    EventLossTable,
    FinancialTerms,
    Layer,
    LayerTerms,
    Trial,
    YearEventTable,
    validate_portfolio,
)


def _f(x: float):
    # JSON has no NaN/inf literals in strict mode: encode them as strings
    x = float(x)
    if math.isnan(x):
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


def _flist(a):
    return [_f(v) for v in np.asarray(a, dtype=np.float64).tolist()]


def dump(name: str, layers, yet) -> dict:
    rep = [str(v) for v in validate_portfolio(layers, yet)]
    return {
        "name": name,
        "catalog": int(yet.catalog_size),
        "ids": np.asarray(yet.event_ids, dtype=np.int64).tolist(),
        "ts": _flist(yet.timestamps),
        "offsets": np.asarray(yet.offsets, dtype=np.int64).tolist(),
        "layers": [{
            "id": str(layer.id),
            "terms": _flist([layer.terms.occ_retention, layer.terms.occ_limit,
                             layer.terms.agg_retention, layer.terms.agg_limit]),
            "elts": [{
                "catalog": int(e.catalog_size),
                "ids": np.asarray(e.event_ids, dtype=np.int64).tolist(),
                "losses": _flist(e.losses),
                "fin": _flist([e.terms.exchange_rate, e.terms.event_retention, e.terms.event_limit,
                               e.terms.share]),
            } for e in layer.elts],
        } for layer in layers],
        "report": rep,
    }


def _small_layer(fin=None, terms=None, cat=10):
    elt = EventLossTable.from_records({4: 100.0, 9: 50.0}, catalog_size=cat, terms=fin)
    return Layer("L", (elt,), terms if terms is not None else LayerTerms())


def _yet(*trials, cat=10):
    return YearEventTable.from_trials([Trial.from_events(*t) for t in trials], catalog_size=cat)


def reference_test_model_cases():
    """pkg/tests/test_model.py:138-258, one case per assertion."""
    ok = _small_layer()
    base = _yet(([4, 9, 4],))
    out = [dump("valid", [ok], base)]
    out.append(dump("no_trials", [ok], YearEventTable(
        10, np.array([], np.uint32), np.array([], np.float64), np.array([0], np.int64))))
    out.append(dump("trial_length_cap", [ok], _yet(([4] * (MAX_TRIAL_LENGTH + 1),))))
    out.append(dump("event_beyond_catalog", [ok], _yet(([11],))))
    out.append(dump("event_id_zero", [ok], _yet(([0],))))
    out.append(dump("timestamp_outside", [ok], _yet(([4, 9], [0.5, 1.5]))))
    out.append(dump("unsorted_within_trial", [ok], _yet(([4, 9], [0.9, 0.1]))))
    out.append(dump("drop_at_boundary", [ok], _yet(([4], [0.9]), ([9], [0.1]))))
    out.append(dump("layer_without_elts", [Layer("empty", (), LayerTerms())], base))
    out.append(dump("negative_layer_terms", [Layer("b", ok.elts, LayerTerms(occ_retention=-1.0))], base))
    out.append(dump("infinite_retention", [Layer("b", ok.elts, LayerTerms(agg_retention=math.inf))], base))
    out.append(dump("zero_limits_legal", [Layer("z", ok.elts, LayerTerms(0.0, 0.0, 0.0, 0.0))], base))
    out.append(dump("catalog_mismatch", [ok], _yet(([4],), cat=99)))
    out.append(dump("duplicate_event", [Layer("d", (EventLossTable(
        10, np.array([4, 4], np.uint32), np.array([1.0, 2.0])),), LayerTerms())], base))
    for i, bad in enumerate((-1.0, math.nan, math.inf)):
        out.append(dump(f"bad_loss_{i}", [Layer("n", (EventLossTable(
            10, np.array([4], np.uint32), np.array([bad])),), LayerTerms())], base))
    for i, ft in enumerate([FinancialTerms(exchange_rate=0.0), FinancialTerms(exchange_rate=math.inf),
                            FinancialTerms(exchange_rate=math.nan), FinancialTerms(event_retention=-1.0),
                            FinancialTerms(event_limit=0.0), FinancialTerms(share=1.5),
                            FinancialTerms(share=-0.1), FinancialTerms(event_retention=math.nan)]):
        out.append(dump(f"bad_fin_{i}", [Layer("f", (EventLossTable(
            10, np.array([4], np.uint32), np.array([1.0]), ft),), LayerTerms())], base))
    bad_elt = EventLossTable(7, np.array([4], np.uint32), np.array([-1.0]), FinancialTerms(share=2.0))
    out.append(dump("report_lists_every_problem", [Layer("multi", (bad_elt,), LayerTerms(occ_limit=-5.0))],
                    _yet(([12],))))
    return out


def repo_host_cases():
    """tests/test_host.py::test_violation_categories and neighbours."""
    ok = _small_layer()
    two = _yet(([4, 9],))
    out = [
        dump("host_out_of_range", [ok], _yet(([99],))),
        dump("host_empty_trial", [ok], _yet(([],))),
        dump("host_bad_ts", [ok], _yet(([4], [1.5]))),
        dump("host_unsorted", [ok], _yet(([4, 9], [0.5, 0.1]))),
        dump("host_elt_out_of_range", [Layer("R", (EventLossTable(
            10, np.array([0, 11], np.uint32), np.array([1.0, 2.0])),), LayerTerms())], two),
        dump("host_layer_nan_terms", [Layer("N", ok.elts, LayerTerms(math.nan, math.nan, math.nan, math.nan))], two),
        dump("host_two_layers", [ok, Layer("M", ok.elts, LayerTerms(occ_limit=-1.0, agg_limit=-2.0))], two),
        dump("host_boundary_drops", [ok], _yet(([4, 9], [0.2, 0.9]), ([4], [0.1]))),
        dump("host_negative_ts", [ok], _yet(([4, 9], [-0.5, 0.2]))),
        dump("host_ts_exact_bounds", [ok], _yet(([4, 9], [0.0, 1.0]))),
    ]
    return out


def device_yet_cases():
    """tests/test_gpu_validate.py::_yet: 30 random trials + injected faults."""
    out = []
    layer = Layer("L", (EventLossTable.from_records({4: 100.0, 9: 50.0}, 50),), LayerTerms(1.0, 60.0, 5.0, 500.0))
    for cases in ["", "range", "zero_id", "empty", "long", "ts_range", "unsorted", "nan",
                  "range empty ts_range unsorted", "long unsorted zero_id", "nan ts_range",
                  "nan unsorted", "empty long range"]:
        rng = np.random.default_rng(5)
        cat = 50
        trials = [Trial.from_events(rng.integers(1, cat + 1, int(rng.integers(1, 40)))) for _ in range(30)]
        if "range" in cases:
            trials[3] = Trial.from_events([1, cat + 1, 2])
        if "zero_id" in cases:
            trials[4] = Trial.from_events([0, 3])
        if "empty" in cases:
            trials[7] = Trial.from_events([])
        if "long" in cases:
            trials[9] = Trial.from_events(np.ones(10_001, dtype=np.int64))
        if "ts_range" in cases:
            trials[2] = Trial.from_events([1, 2], [0.5, 1.5])
        if "unsorted" in cases:
            trials[5] = Trial.from_events([1, 2, 3], [0.1, 0.9, 0.2])
            trials[6] = Trial.from_events([1, 2], [0.8, 0.3])
        if "nan" in cases:
            trials[8] = Trial.from_events([1, 2], [np.nan, 2.0])
        out.append(dump("device_" + (cases.replace(" ", "+") or "clean"), [layer],
                        YearEventTable.from_trials(trials, cat)))
    return out


def random_cases(seed: int, count: int):
    """Seeded mix of every YET- and layer-side fault, several per case."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(count):
        cat = int(rng.integers(5, 400))
        n_trials = int(rng.integers(0, 12))
        trials = []
        for _ in range(n_trials):
            ln = int(rng.integers(0, 25))
            ids = rng.integers(1, cat + 1, ln)
            ts = np.sort(rng.random(ln))
            if ln and rng.random() < 0.15:
                ids[rng.integers(ln)] = rng.choice([0, cat + 1, cat + 7])
            if ln > 1 and rng.random() < 0.15:
                ts = ts[::-1].copy()
            if ln and rng.random() < 0.1:
                ts[rng.integers(ln)] = rng.choice([-0.25, 1.25, np.nan])
            trials.append(Trial.from_events(ids, ts))
        yet = YearEventTable.from_trials(trials, catalog_size=cat)
        layers = []
        for li in range(int(rng.integers(0, 3))):
            elts = []
            for _ in range(int(rng.integers(0, 3))):
                ecat = cat if rng.random() < 0.85 else cat + 1
                n = int(rng.integers(0, 6))
                ids = np.sort(rng.choice(np.arange(1, cat + 1), size=min(n, cat), replace=False)).astype(np.uint32)
                if ids.size and rng.random() < 0.1:
                    ids[-1] = cat + 3
                if ids.size > 1 and rng.random() < 0.1:
                    ids[1] = ids[0]
                losses = rng.lognormal(0, 1, ids.size) * 10
                if ids.size and rng.random() < 0.1:
                    losses[0] = rng.choice([-1.0, np.nan, np.inf])
                fin = [1.0, 0.0, math.inf, 1.0]
                if rng.random() < 0.2:
                    fin[int(rng.integers(4))] = float(rng.choice([-1.0, 0.0, 2.0, np.nan, np.inf]))
                elts.append(EventLossTable(ecat, ids, losses, FinancialTerms(*fin)))
            terms = [0.0, math.inf, 0.0, math.inf]
            if rng.random() < 0.3:
                terms[int(rng.integers(4))] = float(rng.choice([-1.0, np.nan, np.inf, 0.0]))
            layers.append(Layer(f"r{k}_{li}", tuple(elts), LayerTerms(*terms)))
        out.append(dump(f"random_{seed}_{k}", layers, yet))
    return out


def main() -> None:
    cases = reference_test_model_cases() + repo_host_cases() + device_yet_cases() + random_cases(1308, 120)
    with gzip.open(os.path.join(HERE, "validation.json.gz"), "wt") as f:
        json.dump({"generator": "tests/golden/make_validation.py (reference aggrisk.model.validate_portfolio)",
                   "cases": cases}, f, separators=(",", ":"))
    n_bad = sum(1 for c in cases if c["report"])
    print(f"wrote {len(cases)} validation cases ({n_bad} with violations) to {HERE}/validation.json.gz")


if __name__ == "__main__":
    main()
