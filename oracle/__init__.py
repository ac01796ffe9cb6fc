"""CPU oracle for the aggregate-analysis hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs import this package, and
only as the checker (or the timed CPU baseline) -- never as the product.
The product (paper_1308_2066_b200) has no CPU path and never imports it.

Contents
  * run_trials_port  -- ctypes call into liboracle_trials.so, our C
    restatement of the reference hot loop (ref_trials.c, citing
    pkg/src/aggrisk/engine/_kernel.pyx:17-119 line by line).
  * ref_kernel()     -- the reference's OWN Cython kernel, compiled from
    /root/reference/pkg/src/aggrisk/engine/_kernel.pyx into oracle/_ref by
    oracle/Makefile (None when it was not built).
  * run_layer_cpu    -- the reference's thread-pool driver (_run_layer,
    engine/__init__.py:162-201) around either kernel, for the CPU baseline.
  * pml / tvar / ep_points -- numpy restatement of metrics.py:29-115.

Parity pinning (tests/test_oracle.py): the port and the compiled reference
kernel reproduce the golden vectors written from the reference package by
tests/golden/make_golden.py (worked example 150.0, 1000 random oracle
instances bit-for-bit, the seed-31 determinism digest 5ebdd83b8ee0, the C1
YLT).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle_trials.so")

_port = None
_ref = None


def build() -> None:
    """Compile the port (and, where /root/reference exists, oracle/_ref)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load_port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_LIB):
            build()
        lib = ctypes.CDLL(PORT_LIB)
        P, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
        lib.oracle_run_trials.restype = ctypes.c_longlong
        lib.oracle_run_trials.argtypes = [P, P, P, I, P, I, P, P, P, P, D, D, D, D, I, I, I, P, P, I]
        lib.oracle_financial_terms.restype = D
        lib.oracle_financial_terms.argtypes = [D, D, D, D, D]
        lib.oracle_occurrence_terms.restype = D
        lib.oracle_occurrence_terms.argtypes = [D, D, D]
        _port = lib
    return _port


def run_trials_port(event_ids, offsets, stacked, rows, fin_rate, fin_ret, fin_lim, fin_share,
                    occ_ret, occ_lim, agg_ret, agg_lim, chunk, first_trial, last_trial, out,
                    scratch=None) -> int:
    """Same signature and semantics as the reference run_trials."""
    lib = _load_port()
    c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
    ids, offs = c(event_ids, np.uint32), c(offsets, np.int64)
    stk = c(stacked, np.float64)
    rows = c(rows, np.int64)
    fr, fe, fl, fs = (c(a, np.float64) for a in (fin_rate, fin_ret, fin_lim, fin_share))
    if scratch is None:
        scratch = np.empty(max(int(chunk), 1))
    n = lib.oracle_run_trials(ids.ctypes.data, offs.ctypes.data, stk.ctypes.data, stk.shape[1],
                              rows.ctypes.data, rows.shape[0], fr.ctypes.data, fe.ctypes.data,
                              fl.ctypes.data, fs.ctypes.data, occ_ret, occ_lim, agg_ret, agg_lim,
                              int(chunk), int(first_trial), int(last_trial), out.ctypes.data,
                              scratch.ctypes.data, scratch.shape[0])
    if n < 0:
        raise ValueError("oracle: bad run_trials arguments")
    return int(n)


def financial_terms(loss, rate, ret, lim, share) -> float:
    return _load_port().oracle_financial_terms(loss, rate, ret, lim, share)


def occurrence_terms(loss, occ_ret, occ_lim) -> float:
    return _load_port().oracle_occurrence_terms(loss, occ_ret, occ_lim)


def ref_kernel():
    """The reference's compiled Cython run_trials module, or None."""
    global _ref
    if _ref is None:
        found = sorted(glob.glob(os.path.join(HERE, "_ref", "_kernel*.so")))
        if not found:
            return None
        spec = importlib.util.spec_from_file_location("_kernel", found[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _ref = mod
    return _ref


def dense_tables(elts, catalog_size: int) -> np.ndarray:
    """TableSet.from_elts's dense (J, catalog+1) float64 stack (tables.py:107-115)."""
    stacked = np.zeros((len(elts), catalog_size + 1), dtype=np.float64)
    for i, e in enumerate(elts):
        stacked[i, np.asarray(e.event_ids, dtype=np.int64)] = e.losses
    return stacked


def split_by_events(offsets, parts):
    """engine/__init__.py:151-159 (used only to drive the CPU baseline)."""
    n = offsets.shape[0] - 1
    parts = max(1, min(parts, n))
    total = int(offsets[-1])
    cuts = np.searchsorted(offsets, [round(total * k / parts) for k in range(1, parts)], side="left")
    b = sorted({0, n, *map(int, cuts)})
    return [(b[i], b[i + 1]) for i in range(len(b) - 1) if b[i] < b[i + 1]]


def run_layer_cpu(event_ids, offsets, stacked, fin, terms, workers: int = 1, kernel: str = "reference",
                  first: int = 0, last: int | None = None) -> tuple[np.ndarray, int]:
    """The reference _run_layer driver (engine/__init__.py:162-201) over
    trials [first, last): worker_count*4 occurrence-balanced batches on a
    thread pool; `kernel` = "reference" (oracle/_ref) or "port"."""
    last = offsets.shape[0] - 1 if last is None else last
    rows = np.arange(stacked.shape[0], dtype=np.int64)
    rate, ret, lim, share = (np.ascontiguousarray(a, dtype=np.float64) for a in fin)
    out = np.zeros(offsets.shape[0] - 1, dtype=np.float64)
    mod = ref_kernel() if kernel == "reference" else None
    if kernel == "reference" and mod is None:
        raise RuntimeError("oracle/_ref was not built")
    occ_ret, occ_lim, agg_ret, agg_lim = terms

    def task(t0, t1):
        if mod is not None:
            return mod.run_trials(event_ids, offsets, stacked, rows, rate, ret, lim, share,
                                  occ_ret, occ_lim, agg_ret, agg_lim, 0, t0, t1, out, np.empty(1))
        return run_trials_port(event_ids, offsets, stacked, rows, rate, ret, lim, share,
                               occ_ret, occ_lim, agg_ret, agg_lim, 0, t0, t1, out)

    if workers == 1:
        return out, task(first, last)
    sub = offsets[first:last + 1] - offsets[first]
    batches = [(first + a, first + b) for a, b in split_by_events(sub, workers * 4)]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        counts = list(ex.map(lambda b: task(*b), batches))
    return out, sum(counts)


# ---------------------------------------------------------------- metrics --

def order_stat_k(n: int, rp: float) -> int:
    """metrics.py:29-42."""
    rp = float(rp)
    if not rp > 1.0 or rp > n:
        raise ValueError("bad return period")
    return n - math.floor(n / rp)


def pml(losses, rp: float) -> float:
    """metrics.py:45-52 -- np.partition order statistic."""
    a = np.asarray(losses, dtype=np.float64)
    k = order_stat_k(a.shape[0], rp)
    return float(np.partition(a, k - 1)[k - 1])


def tvar(losses, rp: float) -> float:
    """metrics.py:55-63 -- mean of the closed tail."""
    a = np.asarray(losses, dtype=np.float64)
    k = order_stat_k(a.shape[0], rp)
    return float(np.mean(np.partition(a, k - 1)[k - 1:]))


def ep_points(losses, rps) -> tuple:
    """metrics.py:97-115 -- one full sort, (pml, 1/rp) per distinct rp."""
    a = np.sort(np.asarray(losses, dtype=np.float64))
    return tuple((float(a[order_stat_k(a.shape[0], rp) - 1]), 1.0 / rp) for rp in sorted({float(r) for r in rps}))
