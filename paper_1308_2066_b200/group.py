"""Multi-GPU execution through the C ABI: `worker_count` -> a group of GPUs.

The reference parallelises one layer by cutting the trials into contiguous,
occurrence-balanced ranges (`_split_by_events`, pkg/src/aggrisk/engine/
__init__.py:151-159) and running `run_trials` on a thread pool over them
(:193-200).  Here `EngineConfig(worker_count=G)` puts those ranges on up to G
GPUs instead: the partition is `split_by_events(offsets, G)` -- the
reference's own rule, so the trial -> GPU assignment is bit-exact -- the
tables are replicated on every GPU, and ONE library call
(`are_run_layer` / `are_run_layer_host`) runs K2 on all of them.  Each trial
is computed by one warp on one GPU, so the YLT is bit-identical for any G.

`ShardedYearEventTable` is the HBM-resident form: one upload per shard, K0
validation on each GPU, every later layer run over the resident ids.

The group's GPUs default to CUDA devices 0..G-1 (G = min(worker_count, the
visible device count)).  `ARE_GROUP_DEVICES="0,0,0"` pins an explicit member
list -- the same GPU may repeat, which runs several shards on one device and
lets the multi-shard path be exercised on a one-GPU machine.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native
from .portfolio import MAX_TRIAL_LENGTH, Violation

_lock = threading.Lock()
_current: tuple[int, ...] | None = None


def visible_devices() -> int:
    n = ctypes.c_int(0)
    _native.check(_native.load().are_device_count(ctypes.byref(n)))
    return int(n.value)


def devices_for(worker_count: int) -> tuple[int, ...]:
    """The group members a request with `worker_count` workers runs on."""
    env = os.environ.get("ARE_GROUP_DEVICES")
    if env:
        devs = tuple(int(x) for x in env.split(",") if x.strip())
        return devs[: max(1, int(worker_count))] if int(worker_count) < len(devs) else devs
    return tuple(range(max(1, min(int(worker_count), visible_devices()))))


def ensure_group(devices: tuple[int, ...]) -> None:
    """(Re)initialise the library's device group when it differs."""
    global _current
    with _lock:
        if _current == devices:
            return
        arr = (ctypes.c_int * len(devices))(*devices)
        _native.check(_native.load().are_init_devices(arr, len(devices)))
        _current = devices


def shard_bounds(offsets: np.ndarray, parts: int) -> np.ndarray:
    """Trial cut points [0, ..., T] of the reference partition rule."""
    from .engine import split_by_events

    ranges = split_by_events(offsets, parts)
    n = int(offsets.shape[0]) - 1
    if not ranges:
        return np.array([0, n], dtype=np.int64)
    return np.array([r[0] for r in ranges] + [ranges[-1][1]], dtype=np.int64)


def plans_for(tset, devices, rows, rate, ret, lim, share, precombine: bool = False) -> list:
    """One plan per group member (tables replicated to each member's GPU)."""
    return [tset.plan(rows, rate, ret, lim, share, precombine=precombine, device=d) for d in devices]


def _plan_array(plans) -> ctypes.Array:
    return (ctypes.c_void_p * len(plans))(*[p.value for p in plans])


def violations_from_report(r: dict, n_trials: int, n_ids: int, catalog: int) -> list[Violation]:
    """The YET half of validate_portfolio (model.py:371-395) from K0 counters."""
    out = []
    if n_trials == 0:
        out.append(Violation("no_trials", "year event table holds no trials"))
    if r["bad_trials"]:
        out.append(Violation("trial_length", f"{r['bad_trials']} trial(s) outside [1, {MAX_TRIAL_LENGTH}] "
                                             f"occurrences (first: trial {r['first_bad']})"))
    if n_ids:
        if r["min_id"] < 1 or r["max_id"] > catalog:
            out.append(Violation("event_out_of_range", f"trial event id outside [1, {catalog}]"))
        # numpy's min/max propagate NaN, and a NaN compares false: no violation
        if r.get("ts_checked") and not r["ts_nan"] and r["ts_min"] is not None and \
                (r["ts_min"] < 0.0 or r["ts_max"] > 1.0):
            out.append(Violation("bad_timestamp", "timestamps must lie in [0, 1]"))
        if r["unsorted"]:
            out.append(Violation("trial_unsorted", f"timestamps decrease inside {r['unsorted']} position(s)"))
    return out


class ShardedYearEventTable:
    """A YET sharded over a GPU group (trial ranges of the reference rule),
    ids/offsets resident in each member's HBM, validated there by K0."""

    def __init__(self, yet, devices: tuple[int, ...], validate_timestamps: bool = True):
        ensure_group(tuple(devices))
        self.devices = tuple(devices)
        self.catalog_size = int(yet.catalog_size)
        self.offsets = np.ascontiguousarray(yet.offsets, dtype=np.int64)
        self.host = yet
        ids = np.ascontiguousarray(yet.event_ids, dtype=np.uint32)
        ts = getattr(yet, "timestamps", None) if validate_timestamps else None
        ts = None if ts is None else np.ascontiguousarray(ts, dtype=np.float64)
        self.bounds = shard_bounds(self.offsets, len(self.devices))
        h = _native._P()
        _native.check(_native.load().are_yet_upload(
            ids.ctypes.data, ids.shape[0], self.offsets.ctypes.data, self.trial_count,
            None if ts is None else ts.ctypes.data, self.bounds.ctypes.data, self.bounds.size - 1,
            MAX_TRIAL_LENGTH, ctypes.byref(h)))
        self._h = _native.Handle(h.value, "are_yet_free")
        rep = _native.YetReport()
        _native.check(_native.load().are_yet_report(self._h.value, ctypes.byref(rep)))
        self._report = {"min_id": int(rep.min_id), "max_id": int(rep.max_id), "bad_trials": int(rep.bad_trials),
                        "first_bad": int(rep.first_bad_trial), "unsorted": int(rep.unsorted),
                        "ts_nan": int(rep.ts_nan), "ts_min": float(rep.ts_min), "ts_max": float(rep.ts_max),
                        "ts_checked": bool(rep.ts_checked)}
        n_ids = int(self.offsets[-1])
        if rep.ts_checked and int(rep.ts_nan) >= n_ids:
            self._report["ts_min"] = None
        self.ids_validated = n_ids == 0 or int(rep.max_id) <= self.catalog_size

    @property
    def trial_count(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def n_shards(self) -> int:
        return int(self.bounds.size - 1)

    @property
    def event_ids(self) -> np.ndarray:
        return self.host.event_ids

    @property
    def timestamps(self):
        return getattr(self.host, "timestamps", None)

    def yet_violations(self) -> list[Violation]:
        return violations_from_report(self._report, self.trial_count, int(self.offsets[-1]), self.catalog_size)

    def run_layer(self, plans, terms, out: np.ndarray | None, variant: str = "auto", rps=None,
                  first: int = 0, last: int | None = None):
        """K2 on every shard's GPU (one library call); returns lookups, or
        (lookups, pml, tvar) when return periods are given (K3 on the
        gathered table)."""
        last = self.trial_count if last is None else int(last)
        flags = _native.IDS_VALIDATED if self.ids_validated and all(
            _native.plan_info(p).row_len > int(self._report["max_id"]) for p in plans[:1]) else 0
        lookups = _native._I64()
        rp = None if rps is None else np.ascontiguousarray(rps, dtype=np.float64)
        n_rp = 0 if rp is None else rp.size
        pml = np.empty(max(n_rp, 1))
        tvar = np.empty(max(n_rp, 1))
        _native.check(_native.load().are_run_layer(
            self._h.value, _plan_array(plans), len(plans), float(terms.occ_retention), float(terms.occ_limit),
            float(terms.agg_retention), float(terms.agg_limit), int(first), last,
            None if out is None else out.ctypes.data, ctypes.byref(lookups), _native.VARIANTS[variant] | flags,
            None if rp is None else rp.ctypes.data, n_rp, pml.ctypes.data, tvar.ctypes.data))
        if rp is None:
            return int(lookups.value)
        return int(lookups.value), pml[:n_rp], tvar[:n_rp]

    def close(self) -> None:
        self._h.close()


def run_layer_host(yet, plans, bounds: np.ndarray, terms, out: np.ndarray, variant: str = "auto",
                   validated: bool = False) -> int:
    """Host-resident YET on a group: shard s streams its trials to its GPU
    over that GPU's PCIe link, all shards concurrently (one library call)."""
    ids = np.ascontiguousarray(yet.event_ids, dtype=np.uint32)
    offs = np.ascontiguousarray(yet.offsets, dtype=np.int64)
    n = int(offs.shape[0]) - 1
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    lookups = _native._I64()
    _native.check(_native.load().are_run_layer_host(
        ids.ctypes.data, ids.shape[0], offs.ctypes.data, n, b.ctypes.data, b.size - 1, _plan_array(plans),
        float(terms.occ_retention), float(terms.occ_limit), float(terms.agg_retention), float(terms.agg_limit),
        0, n, out.ctypes.data, ctypes.byref(lookups),
        _native.VARIANTS[variant] | (_native.IDS_VALIDATED if validated else 0)))
    return int(lookups.value)
