"""Device-resident direct-access tables (K1 host side).

Mirrors the reference's `TableSet` / `DirectAccessTable` API
(pkg/src/aggrisk/tables.py:45-198): same constructors, the same
`selection_arrays` contract (selection order = accumulation order,
tables.py:133-153), the same memory accounting (8-byte slots, slot 0 as
overhead, tables.py:184-198) and the same build counter (tables.py:29-42).

What changes is where the tables live.  `TableSet.from_elts` uploads the
sparse ELT records and scatters them into dense float64 rows ON THE DEVICE
(K1, csrc/k1_ingest.cu); the host never materialises the (J, catalog+1)
array unless `.stacked` is read.  For every (selection, financial terms)
the set builds -- once, cached -- a hot-set plan on the device: the 16-byte
per-event records and the shared-memory filter K2 runs on.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .errors import EventOutOfRangeError
from .portfolio import FinancialTerms

BYTES_PER_SLOT = 8
_PLAN_CACHE = 8

_builds = 0
_builds_lock = threading.Lock()


def build_count() -> int:
    """TableSet builds since import (reference tables.py:33-36)."""
    return _builds


def _count_build() -> None:
    global _builds
    with _builds_lock:
        _builds += 1


class DirectAccessTable:
    """One dense table viewed from the host; `losses` is fetched lazily."""

    __slots__ = ("catalog_size", "terms", "nonzero_count", "_owner", "_row", "_losses")

    def __init__(self, catalog_size: int, losses, terms: FinancialTerms, nonzero_count: int,
                 _owner: "TableSet | None" = None, _row: int = 0):
        self.catalog_size = int(catalog_size)
        self.terms = terms
        self.nonzero_count = int(nonzero_count)
        self._owner, self._row = _owner, _row
        self._losses = None
        if losses is not None:
            self._losses = np.ascontiguousarray(losses, dtype=np.float64)
            self._losses.setflags(write=False)

    @property
    def losses(self) -> np.ndarray:
        if self._losses is None:
            self._losses = self._owner.stacked[self._row]
        return self._losses

    def lookup(self, event: int) -> float:
        if not 1 <= event <= self.catalog_size:
            raise EventOutOfRangeError(f"event id {event} outside [1, {self.catalog_size}]")
        return float(self.losses[event])

    def __repr__(self) -> str:
        return f"DirectAccessTable(catalog={self.catalog_size}, nonzero={self.nonzero_count})"


class TableSet:
    """The direct-access tables of one layer / session, resident on the B200."""

    __slots__ = ("catalog_size", "tables", "fin_rate", "fin_ret", "fin_lim", "fin_share",
                 "_dev", "_stacked", "_plans", "_lock", "_replicas", "__weakref__")

    def __init__(self, catalog_size: int, stacked, terms: Sequence[FinancialTerms],
                 nonzero: Sequence[int], *, _device_tables=None):
        """Reference-compatible constructor: dense (n, catalog+1) float64 rows."""
        self.catalog_size = int(catalog_size)
        terms = list(terms)
        self._stacked = None
        if stacked is not None:
            self._stacked = np.ascontiguousarray(stacked, dtype=np.float64)
            self._stacked.setflags(write=False)
        self._dev = _device_tables if _device_tables is not None else _native.tables_from_dense(
            self._stacked.reshape(len(terms), self.catalog_size + 1))
        self.tables = tuple(
            DirectAccessTable(self.catalog_size, None, t, nz, _owner=self, _row=i)
            for i, (t, nz) in enumerate(zip(terms, nonzero)))
        self.fin_rate = np.array([t.exchange_rate for t in terms], dtype=np.float64)
        self.fin_ret = np.array([t.event_retention for t in terms], dtype=np.float64)
        self.fin_lim = np.array([t.event_limit for t in terms], dtype=np.float64)
        self.fin_share = np.array([t.share for t in terms], dtype=np.float64)
        self._plans: OrderedDict = OrderedDict()
        self._lock = threading.Lock()
        self._replicas: dict[int, _native.Handle] = {}  # device -> copy of the tables (multi-GPU group)
        _count_build()

    @classmethod
    def from_elts(cls, elts: Sequence, catalog_size: int | None = None) -> "TableSet":
        """K1: scatter every ELT into its dense device row (tables.py:95-117)."""
        if catalog_size is None:
            if not elts:
                raise ValueError("catalog_size required for an empty table set")
            catalog_size = max(e.catalog_size for e in elts)
        row_len = int(catalog_size) + 1
        ids, losses, bounds, nonzero = [], [], [0], []
        for i, elt in enumerate(elts):
            e_ids = np.ascontiguousarray(elt.event_ids, dtype=np.uint32)
            e_loss = np.ascontiguousarray(elt.losses, dtype=np.float64)
            if e_ids.size and (int(e_ids.min()) < 1 or int(e_ids.max()) > catalog_size):
                raise EventOutOfRangeError(f"elt[{i}] holds event ids outside [1, {catalog_size}]")
            if e_ids.size > 1 and not np.all(e_ids[1:] > e_ids[:-1]):
                # unsorted or duplicated ids: numpy's last-write-wins scatter
                # semantics (tables.py:115) are reproduced by deduplicating
                # on the host, keeping the last record per id
                rev = e_ids[::-1]
                _, first_in_rev = np.unique(rev, return_index=True)
                keep = e_ids.size - 1 - first_in_rev
                e_ids, e_loss = e_ids[keep], e_loss[keep]
            ids.append(e_ids)
            losses.append(e_loss)
            bounds.append(bounds[-1] + e_ids.size)
            nonzero.append(int(np.count_nonzero(e_loss)))
        dev = _native.tables_from_records(
            np.concatenate(ids) if ids else np.empty(0, np.uint32),
            np.concatenate(losses) if losses else np.empty(0),
            np.asarray(bounds, dtype=np.int64), row_len)
        return cls(catalog_size, None, [e.terms for e in elts], nonzero, _device_tables=dev)

    @classmethod
    def from_tables(cls, tables: Sequence[DirectAccessTable]) -> "TableSet":
        if not tables:
            raise ValueError("need at least one table")
        cat = tables[0].catalog_size
        if any(t.catalog_size != cat for t in tables):
            raise ValueError("tables span different catalogs")
        stacked = np.vstack([t.losses for t in tables])
        return cls(cat, stacked, [t.terms for t in tables], [t.nonzero_count for t in tables])

    def __len__(self) -> int:
        return len(self.tables)

    @property
    def stacked(self) -> np.ndarray:
        """Dense (n, catalog+1) float64 host copy, fetched from the device on demand."""
        if self._stacked is None:
            rows = [_native.read_row(self._dev, i, self.catalog_size + 1) for i in range(len(self.tables))]
            arr = np.vstack(rows) if rows else np.zeros((0, self.catalog_size + 1))
            arr.setflags(write=False)
            self._stacked = arr
        return self._stacked

    @property
    def device_tables(self) -> _native.Handle:
        return self._dev

    def selection_arrays(self, indices: Sequence[int] | None = None):
        """(rows, rate, ret, lim, share) for a subset (tables.py:133-153)."""
        if indices is None:
            sel = np.arange(len(self.tables), dtype=np.int64)
        else:
            sel = np.asarray(list(indices), dtype=np.int64)
            if sel.size == 0:
                raise ValueError("table selection is empty")
            if sel.min() < 0 or sel.max() >= len(self.tables):
                raise IndexError("table selection out of range")
        return (sel, np.ascontiguousarray(self.fin_rate[sel]), np.ascontiguousarray(self.fin_ret[sel]),
                np.ascontiguousarray(self.fin_lim[sel]), np.ascontiguousarray(self.fin_share[sel]))

    @property
    def device(self) -> int:
        """CUDA ordinal holding the tables."""
        return _native.tables_device(self._dev)

    def tables_on(self, device: int) -> _native.Handle:
        """The tables in `device`'s memory: the original, or a peer copy made
        once (the multi-GPU group replicates tables)."""
        if device is None or device == self.device:
            return self._dev
        with self._lock:
            rep = self._replicas.get(device)
            if rep is None:
                rep = self._replicas[device] = _native.tables_replicate(self._dev, device)
            return rep

    def plan(self, rows, rate, ret, lim, share, pool: bool = False, precombine: bool = False,
             device: int | None = None) -> _native.Handle:
        """Device hot set for this selection + financial terms (cached, LRU);
        `pool` sizes it for the fused multi-layer kernel; `precombine` folds
        the financial terms into one value per event;
        `device` builds it on that GPU's replica of the tables.

        An evicted plan is only dropped from the cache, never freed here: a
        caller that still holds it (another thread's K2 launch, the
        reference's concurrent run_trials, engine/__init__.py:195-200) keeps
        it alive, and it is released when the last reference goes."""
        dev = None if device is None or device == self.device else int(device)
        key = (dev, pool, precombine, np.asarray(rows, np.int64).tobytes(),
               np.asarray(rate, np.float64).tobytes(), np.asarray(ret, np.float64).tobytes(),
               np.asarray(lim, np.float64).tobytes(), np.asarray(share, np.float64).tobytes())
        with self._lock:
            hit = self._plans.get(key)
            if hit is not None:
                self._plans.move_to_end(key)
                return hit
        plan = _native.plan_build(self.tables_on(dev), rows, rate, ret, lim, share, pool=pool, precombine=precombine)
        with self._lock:
            self._plans[key] = plan
            while len(self._plans) > _PLAN_CACHE:
                self._plans.popitem(last=False)  # freed by its last holder (Handle.__del__)
        return plan


def build_direct_table(elt) -> DirectAccessTable:
    return TableSet.from_elts([elt], elt.catalog_size).tables[0]


def lookup(table: DirectAccessTable, event: int) -> float:
    return table.lookup(event)


@dataclass(frozen=True)
class MemoryFootprint:
    table_count: int
    payload_slots: int
    payload_bytes: int
    overhead_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.payload_bytes + self.overhead_bytes


def memory_footprint(tables: Sequence[DirectAccessTable]) -> MemoryFootprint:
    """Dense float64 accounting of the direct-access tables (tables.py:184-198)."""
    slots = sum(int(t.catalog_size) for t in tables)
    return MemoryFootprint(len(tables), slots, slots * BYTES_PER_SLOT, len(tables) * BYTES_PER_SLOT)
