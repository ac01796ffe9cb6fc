"""Golden-fixture loaders shared by the CPU and GPU tests.

`load_instances()` unpacks tests/golden/random_instances_1001.npz (written by
tests/golden/make_golden.py from the reference's pkg/tests/oracle.py
random_instance with default_rng(1001), as test_acceptance.py:47-63 does)
into this package's own types, together with the reference engine's YLT and
the reference's naive-oracle YLT for each instance.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from paper_1308_2066_b200.portfolio import (
    EventLossTable,
    FinancialTerms,
    Layer,
    LayerTerms,
    Trial,
    YearEventTable,
)

HERE = os.path.dirname(os.path.abspath(__file__))


@dataclass
class Instance:
    layer: Layer
    yet: YearEventTable
    ylt: np.ndarray          # reference engine output (bit-exact target)
    ylt_naive: np.ndarray    # reference tests/oracle.py layer_ylt output

    @property
    def stacked(self) -> np.ndarray:
        st = np.zeros((len(self.layer.elts), self.yet.catalog_size + 1))
        for i, e in enumerate(self.layer.elts):
            st[i, e.event_ids.astype(np.int64)] = e.losses
        return st

    def fin(self):
        t = [e.terms for e in self.layer.elts]
        return (np.array([x.exchange_rate for x in t]), np.array([x.event_retention for x in t]),
                np.array([x.event_limit for x in t]), np.array([x.share for x in t]))


def load_instances() -> list[Instance]:
    with np.load(os.path.join(HERE, "golden", "random_instances_1001.npz")) as f:
        z = {k: f[k] for k in f.files}  # decompress each array once
    out = []
    e_at = 0
    n_inst = z["catalog"].shape[0]
    for i in range(n_inst):
        cat = int(z["catalog"][i])
        elts = []
        for _ in range(int(z["n_elts"][i])):
            lo, hi = z["elt_offsets"][e_at], z["elt_offsets"][e_at + 1]
            f = z["fin_terms"][e_at]
            elts.append(EventLossTable(cat, z["elt_ids"][lo:hi], z["elt_losses"][lo:hi],
                                       FinancialTerms(*map(float, f))))
            e_at += 1
        lt = LayerTerms(*map(float, z["layer_terms"][i]))
        t0, t1 = int(z["trial_bounds"][i]), int(z["trial_bounds"][i + 1])
        offs = z["trial_offsets"][t0:t1 + 1]
        base = int(offs[0])
        offs = offs - base
        ids = z["event_ids"][base: base + int(offs[-1])]
        # Trial.from_events timestamps (linspace per trial) -- never read by compute
        ts = np.concatenate([np.linspace(0.0, 1.0, int(b - a)) if b - a > 1 else np.zeros(int(b - a))
                             for a, b in zip(offs[:-1], offs[1:])]) if offs.size > 1 else np.zeros(0)
        yet = YearEventTable(cat, ids, ts, offs)
        y0, y1 = int(z["ylt_bounds"][i]), int(z["ylt_bounds"][i + 1])
        out.append(Instance(Layer("oracle", tuple(elts), lt), yet, z["ylt"][y0:y1], z["ylt_naive_oracle"][y0:y1]))
    return out


def trial_from(ids) -> Trial:
    return Trial.from_events(list(ids))
