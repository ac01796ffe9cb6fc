"""Loader for tests/golden/validation.json.gz: reference `validate_portfolio`
reports (model.py:360-404, written by tests/golden/make_validation.py),
rebuilt here with this repo's types."""

from __future__ import annotations

import gzip
import json
import math
import os

import numpy as np

from paper_1308_2066_b200.portfolio import EventLossTable, FinancialTerms, Layer, LayerTerms, YearEventTable
from tests.conftest import GOLDEN

_SPECIAL = {"nan": math.nan, "inf": math.inf, "-inf": -math.inf}


def _f(v):
    return _SPECIAL[v] if isinstance(v, str) else float(v)


def _fa(vs):
    return np.array([_f(v) for v in vs], dtype=np.float64)


def load_cases() -> list[dict]:
    with gzip.open(os.path.join(GOLDEN, "validation.json.gz"), "rt") as f:
        return json.load(f)["cases"]


def build(case: dict):
    """(layers, yet) of one case, as this repo's objects."""
    yet = YearEventTable(case["catalog"], np.array(case["ids"], dtype=np.uint32), _fa(case["ts"]),
                         np.array(case["offsets"], dtype=np.int64))
    layers = []
    for lay in case["layers"]:
        elts = tuple(EventLossTable(e["catalog"], np.array(e["ids"], dtype=np.uint32), _fa(e["losses"]),
                                    FinancialTerms(*[_f(v) for v in e["fin"]])) for e in lay["elts"])
        layers.append(Layer(lay["id"], elts, LayerTerms(*[_f(v) for v in lay["terms"]])))
    return layers, yet
