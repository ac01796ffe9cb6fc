"""Session-resident re-pricing on the GPU.

Mirrors the reference pricing service's session semantics
(pkg/src/aggrisk/service.py:113-241): a session pins a year event table and
the direct-access tables of an ELT pool; each reprice runs the engine with new
layer terms over an optional ELT subset and reports PML/TVaR per return period,
the EP curve, mean and max.  Here the YET ids live in HBM
(`DeviceYearEventTable`), the tables and every (selection, terms) hot-set plan
stay on the device, the YLT never leaves HBM, and PML/TVaR/EP come from one K3
call -- so a reprice is K2 + K3, with no PCIe traffic except the scalars.
Tables are built once per session (`build_count` does not move on reprice,
test_service.py:264-282).
"""

from __future__ import annotations

import time
from typing import Sequence

import numpy as np

from .direct_access import TableSet
from .errors import PortfolioInvalidError
from .portfolio import Layer, LayerTerms, validate_portfolio
from .resident import DeviceYearEventTable
from .risk import _order_stat_k, order_stats_summary, pml_many

DEFAULT_RETURN_PERIODS = (10.0, 50.0, 100.0, 250.0)  # service.py:45


class PricingSession:
    def __init__(self, yet, elts: Sequence, validate: bool = True):
        import torch

        self.yet = yet if isinstance(yet, DeviceYearEventTable) else DeviceYearEventTable(yet)
        if validate:  # service.py:180-186: the whole pool is validated once
            violations = validate_portfolio([Layer("session", tuple(elts), LayerTerms())], self.yet)
            if violations:
                raise PortfolioInvalidError(violations)
        self.tset = TableSet.from_elts(list(elts), self.yet.catalog_size)
        self.d_ylt = torch.empty(self.yet.trial_count, dtype=torch.float64, device=self.yet.device)
        self.reprice_count = 0
        self.created_at = time.time()

    def reprice(self, terms: LayerTerms, selection: Sequence[int] | None = None,
                return_periods: Sequence[float] = DEFAULT_RETURN_PERIODS) -> dict:
        """service.py:213-241 on the device; same result keys."""
        import torch

        n = self.yet.trial_count
        rps = [float(r) for r in return_periods]
        for r in rps:
            _order_stat_k(n, r)  # reference argument errors before any work
        rows, rate, ret, lim, share = self.tset.selection_arrays(selection)
        plan = self.tset.plan(rows, rate, ret, lim, share)
        torch.cuda.synchronize(self.yet.device)
        t0 = time.perf_counter()
        self.yet.simulate_device(plan, terms, out=self.d_ylt)
        distinct = sorted(set(rps))
        # one K3 call: PML/TVaR, the EP points and the mean/max from its tail
        # pass (many EP points: one device sort instead)
        if len(rps) + len(distinct) <= 8:
            p, t, mean, peak = order_stats_summary(self.d_ylt, rps + distinct)
            ep = p[len(rps):]
        else:
            p, t, mean, peak = order_stats_summary(self.d_ylt, rps)
            ep = pml_many(self.d_ylt, distinct)
        engine_seconds = time.perf_counter() - t0
        self.reprice_count += 1
        return {
            "trial_count": n,
            "metrics": [{"return_period": rp, "pml": float(p[i]), "tvar": float(t[i])} for i, rp in enumerate(rps)],
            "ep_curve": [{"loss": float(ep[i]), "exceedance_probability": 1.0 / rp}
                         for i, rp in enumerate(distinct)],
            "trial_mean": mean,
            "trial_max": peak,
            "lookups": int(rows.shape[0]) * int(self.yet.offsets[-1]),
            "engine_seconds": engine_seconds,
        }

    def losses(self) -> np.ndarray:
        """The last reprice's YLT, copied to the host."""
        return self.d_ylt.cpu().numpy()
