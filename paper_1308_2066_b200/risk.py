"""Tail metrics over Year Loss Tables, computed by K3 on the GPU.

Mirrors pkg/src/aggrisk/metrics.py: `pml`, `tvar`, `ep_curve`, `EPCurve`,
`portfolio_rollup`, with the same rank rule k = n - floor(n / rp)
(metrics.py:29-42), the same argument errors, and the closed-tail TVaR.
`order_stats` evaluates many return periods in one device pass (the pricing
service asks for four at a time, service.py:223-227).

Inputs may be a YearLossTable, a numpy array (copied to the device), or a
float64 CUDA tensor already in HBM (no copy).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _native
from .portfolio import YearLossTable


def _order_stat_k(n: int, return_period: float) -> int:
    rp = float(return_period)
    if not rp > 1.0:
        raise ValueError(f"return_period must exceed 1, got {return_period}")
    if rp > n:
        raise ValueError(f"return_period {return_period} exceeds trial count {n}")
    return n - math.floor(n / rp)


def _check_rps(n: int, rps: np.ndarray) -> None:
    """_order_stat_k's checks for every return period at once; the first
    offending one raises the reference's message."""
    bad = ~(rps > 1.0) | (rps > n)
    if bad.any():
        _order_stat_k(n, float(rps[int(np.argmax(bad))]))


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _source(ylt):
    losses = ylt.losses if isinstance(ylt, YearLossTable) or hasattr(ylt, "layer_id") else ylt
    if _is_cuda_tensor(losses):
        if losses.dim() != 1:
            raise ValueError("losses must be one-dimensional")
        return losses.contiguous().double()
    arr = np.ascontiguousarray(losses, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError("losses must be one-dimensional")
    return arr


def order_stats(ylt, return_periods: Sequence[float], stream=None) -> tuple[np.ndarray, np.ndarray]:
    """(pml[r], tvar[r]) for every return period, one K3 launch sequence."""
    src = _source(ylt)
    n = int(src.shape[0])
    if n == 0:
        raise ValueError("empty year loss table")
    rps = np.ascontiguousarray([float(r) for r in return_periods], dtype=np.float64)
    _check_rps(n, rps)
    pml_out = np.empty(rps.size)
    tvar_out = np.empty(rps.size)
    if rps.size == 0:
        return pml_out, tvar_out
    lib = _native.load()
    if _is_cuda_tensor(src):
        import torch

        st = torch.cuda.current_stream(src.device) if stream is None else stream
        _native.check(lib.are_order_stats_device(src.data_ptr(), n, rps.ctypes.data, rps.size,
                                                 pml_out.ctypes.data, tvar_out.ctypes.data,
                                                 ctypes.c_void_p(st.cuda_stream)))
    else:
        _native.check(lib.are_order_stats_host(src.ctypes.data, n, rps.ctypes.data, rps.size,
                                               pml_out.ctypes.data, tvar_out.ctypes.data))
    return pml_out, tvar_out


# Above this many return periods a PML-only request (an EP curve) sorts the
# table once on the device (are_pml_many_device) instead of running the
# select kernel once per 8 return periods.
SORT_MIN_RPS = 9


def pml_many(ylt, return_periods: Sequence[float], stream=None) -> np.ndarray:
    """PML at every return period (no TVaR): one device sort + one gather
    when there are many, the select kernel otherwise."""
    src = _source(ylt)
    n = int(src.shape[0])
    if n == 0:
        raise ValueError("empty year loss table")
    rps = np.ascontiguousarray(return_periods, dtype=np.float64).reshape(-1)
    _check_rps(n, rps)
    if rps.size < SORT_MIN_RPS:
        return order_stats(src, rps, stream)[0]
    import torch

    d = src if _is_cuda_tensor(src) else torch.from_numpy(src).cuda()
    out = np.empty(rps.size)
    st = torch.cuda.current_stream(d.device) if stream is None else stream
    with torch.cuda.device(d.device):
        _native.check(_native.load().are_pml_many_device(d.data_ptr(), n, rps.ctypes.data, rps.size, out.ctypes.data,
                                                         ctypes.c_void_p(st.cuda_stream)))
    return out


def order_stats_async(d_ylt, return_periods: Sequence[float], d_res, stream, max_ctas: int = 0) -> None:
    """K3 without a host wait, for pipelined callers: pml[r] lands in d_res[r]
    and tvar[r] in d_res[8 + r] (a float64 CUDA tensor of >= 16), ordered on
    `stream`; at most `max_ctas` CTAs (0: the full grid).  One stream per
    device for every asynchronous call (they share a workspace)."""
    n = int(d_ylt.shape[0])
    if n == 0:
        raise ValueError("empty year loss table")
    rps = np.ascontiguousarray([float(r) for r in return_periods], dtype=np.float64)
    _check_rps(n, rps)
    if not 1 <= rps.size <= 8:
        raise ValueError("order_stats_async takes 1..8 return periods")
    import torch

    if d_res.dtype != torch.float64 or d_res.numel() < 16:
        raise ValueError("d_res must be a float64 CUDA tensor of at least 16 values")
    _native.check(_native.load().are_order_stats_async(d_ylt.data_ptr(), n, rps.ctypes.data, rps.size,
                                                       d_res.data_ptr(), int(max_ctas),
                                                       ctypes.c_void_p(stream.cuda_stream)))


def order_stats_summary(d_ylt, return_periods: Sequence[float], stream=None):
    """(pml, tvar, mean, max) from one K3 call over a float64 CUDA tensor: the
    mean and maximum ride along in the tail pass (the pricing service's
    trial_mean / trial_max, service.py:237-238)."""
    import torch

    n = int(d_ylt.shape[0])
    if n == 0:
        raise ValueError("empty year loss table")
    rps = np.ascontiguousarray([float(r) for r in return_periods], dtype=np.float64)
    _check_rps(n, rps)
    pml_out = np.empty(max(rps.size, 1))
    tvar_out = np.empty(max(rps.size, 1))
    mm = np.empty(2)
    st = torch.cuda.current_stream(d_ylt.device) if stream is None else stream
    _native.check(_native.load().are_order_stats_summary_device(
        d_ylt.data_ptr(), n, rps.ctypes.data, rps.size, pml_out.ctypes.data, tvar_out.ctypes.data, mm.ctypes.data,
        ctypes.c_void_p(st.cuda_stream)))
    return pml_out[:rps.size], tvar_out[:rps.size], float(mm[0]), float(mm[1])


def pml(ylt, return_period: float) -> float:
    """Probable maximum loss at `return_period` (metrics.py:45-52)."""
    return float(order_stats(ylt, [return_period])[0][0])


def tvar(ylt, return_period: float) -> float:
    """Mean of the losses at and beyond the PML order statistic (metrics.py:55-63)."""
    return float(order_stats(ylt, [return_period])[1][0])


@dataclass(frozen=True)
class EPCurve:
    """(loss, exceedance probability) points, probabilities strictly decreasing."""

    points: tuple

    def __post_init__(self):
        pts = tuple(tuple(p) for p in self.points)
        object.__setattr__(self, "points", pts)
        for (l0, p0), (l1, p1) in zip(pts, pts[1:]):
            if not p1 < p0:
                raise ValueError("probabilities must be strictly decreasing")
            if l1 < l0:
                raise ValueError("losses must be non-decreasing")
        if any(not 0.0 <= p <= 1.0 for _, p in pts):
            raise ValueError("probability outside [0, 1]")

    @classmethod
    def _from_arrays(cls, loss: np.ndarray, prob: np.ndarray) -> "EPCurve":
        """The same invariants checked on arrays (first failing pair first),
        for curves built from one device pass: no per-point Python loop."""
        p_bad = ~(prob[1:] < prob[:-1])
        l_bad = loss[1:] < loss[:-1]
        if p_bad.any() or l_bad.any():
            ip = int(np.argmax(p_bad)) if p_bad.any() else prob.size
            il = int(np.argmax(l_bad)) if l_bad.any() else prob.size
            raise ValueError("probabilities must be strictly decreasing" if ip <= il else "losses must be non-decreasing")
        if not np.all((prob >= 0.0) & (prob <= 1.0)):
            raise ValueError("probability outside [0, 1]")
        self = object.__new__(cls)
        object.__setattr__(self, "points", tuple(zip(loss.tolist(), prob.tolist())))
        return self

    @property
    def losses(self) -> tuple:
        return tuple(l for l, _ in self.points)

    @property
    def probabilities(self) -> tuple:
        return tuple(p for _, p in self.points)

    def __len__(self) -> int:
        return len(self.points)

    def __iter__(self):
        return iter(self.points)


def ep_curve(ylt, return_periods: Iterable[float]) -> EPCurve:
    """PML at each distinct return period, ascending rp (metrics.py:97-115)."""
    src = _source(ylt)
    if int(src.shape[0]) == 0:
        raise ValueError("empty year loss table")
    rps = sorted({float(r) for r in return_periods})
    if not rps:
        raise ValueError("no return periods given")
    rp_arr = np.asarray(rps, dtype=np.float64)
    p = pml_many(src, rp_arr)
    return EPCurve._from_arrays(np.asarray(p, dtype=np.float64), 1.0 / rp_arr)


def portfolio_rollup(ylts: Sequence[YearLossTable]) -> YearLossTable:
    """Per-trial sum across layers in list order (metrics.py:118-133), on the GPU."""
    if not ylts:
        raise ValueError("no year loss tables to roll up")
    if len(ylts) == 1:
        return ylts[0]
    n = ylts[0].losses.shape[0]
    for y in ylts[1:]:
        if y.losses.shape[0] != n:
            raise ValueError(f"year loss tables differ in length: {n} vs {y.losses.shape[0]}")
    import torch

    dev = [torch.as_tensor(np.ascontiguousarray(y.losses, dtype=np.float64)).cuda() for y in ylts]
    total = rollup_device(dev)
    return YearLossTable("portfolio", total.cpu().numpy())


def rollup_device(tensors, out=None, stream=None):
    """d_out[t] = ((y0[t] + y1[t]) + ...) for float64 CUDA tensors (K3 roll-up)."""
    import torch

    n = int(tensors[0].shape[0])
    out = torch.empty(n, dtype=torch.float64, device=tensors[0].device) if out is None else out
    ptrs = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    st = torch.cuda.current_stream(tensors[0].device) if stream is None else stream
    _native.check(_native.load().are_rollup_device(ctypes.cast(ptrs, ctypes.c_void_p), len(tensors), n, out.data_ptr(),
                                                   ctypes.c_void_p(st.cuda_stream)))
    return out
