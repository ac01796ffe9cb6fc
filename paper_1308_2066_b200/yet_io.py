"""ARE1 binary Year Event Tables: read (host, ids-only, or straight into HBM)
and write, in the reference's format (pkg/src/aggrisk/io.py:150-201).

Layout of a YET file: ``ARE1`` magic, <u16 version, u16 kind>, <u64 catalog,
u64 trials, u64 occurrences>, then int64 offsets[trials+1], uint32
ids[occurrences], float64 timestamps[occurrences].  The ids therefore sit at
byte offset 32 + 8 * (trials + 1).

`load_yet_device` is §8(f) row 1's direct ids-only load: the ids and offsets
are memory-mapped and copied to the GPU in chunks; the timestamps (2/3 of the
file, never read by the simulation) are streamed through the
device validator (K0) and dropped instead of being materialised on the host.
Errors are the reference's: FormatMismatchError, VersionMismatchError,
TruncatedPayloadError, DataFormatError (io.py:63-112).
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .errors import DataFormatError, FormatMismatchError, TruncatedPayloadError, VersionMismatchError
from .portfolio import YearEventTable

MAGIC = b"ARE1"
VERSION = 1
KIND_YET = 1
_KINDS = {1: "yet", 2: "elt", 3: "layer", 4: "ylt"}
_HEADER = 32


def _header(path: str):
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(_HEADER)
    if len(head) < 8 or head[:4] != MAGIC:
        raise FormatMismatchError(f"{path}: bad magic {head[:4]!r}, expected {MAGIC!r}")
    version, kind = struct.unpack("<HH", head[4:8])
    if version != VERSION:
        raise VersionMismatchError(f"{path}: format version {version}, this build reads {VERSION}")
    if kind not in _KINDS:
        raise FormatMismatchError(f"{path}: unknown kind code {kind}")
    if kind != KIND_YET:
        raise FormatMismatchError(f"{path}: holds a {_KINDS[kind]}, expected a yet")
    if len(head) < _HEADER:
        raise TruncatedPayloadError(f"{path}: needed 24 bytes at offset 8, file has {size}")
    catalog, trials, total = struct.unpack("<QQQ", head[8:32])
    need = _HEADER + 8 * (trials + 1) + 12 * total
    if size < need:
        raise TruncatedPayloadError(f"{path}: needed {need} bytes, file has {size}")
    if size > need:
        raise DataFormatError(f"{path}: {size - need} trailing bytes")
    return int(catalog), int(trials), int(total)


def _maps(path: str, trials: int, total: int):
    offsets = np.memmap(path, dtype=np.int64, mode="r", offset=_HEADER, shape=(trials + 1,))
    ids_at = _HEADER + 8 * (trials + 1)
    ids = np.memmap(path, dtype=np.uint32, mode="r", offset=ids_at, shape=(total,)) if total else \
        np.zeros(0, np.uint32)
    ts = np.memmap(path, dtype=np.float64, mode="r", offset=ids_at + 4 * total, shape=(total,)) if total else \
        np.zeros(0)
    if offsets.shape[0] and (offsets[0] != 0 or offsets[-1] != total):
        raise DataFormatError(f"{path}: offset vector inconsistent with payload")
    return offsets, ids, ts


def load_yet(path, ids_only: bool = False) -> YearEventTable:
    """Host YearEventTable from an ARE1 file (ids_only: skip the timestamps)."""
    path = os.fspath(path)
    catalog, trials, total = _header(path)
    offsets, ids, ts = _maps(path, trials, total)
    return YearEventTable(catalog, np.array(ids), None if ids_only else np.array(ts), np.array(offsets))


def save_yet(yet, path) -> None:
    """Write `yet` in the reference's ARE1 binary layout (io.py:150-160)."""
    total = int(yet.offsets[-1])
    ts = yet.timestamps if yet.timestamps is not None else np.zeros(total)
    with open(os.fspath(path), "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<HH", VERSION, KIND_YET))
        f.write(struct.pack("<QQQ", yet.catalog_size, yet.trial_count, total))
        f.write(np.ascontiguousarray(yet.offsets, dtype=np.int64).tobytes())
        f.write(np.ascontiguousarray(yet.event_ids, dtype=np.uint32).tobytes())
        f.write(np.ascontiguousarray(ts, dtype=np.float64).tobytes())


def load_yet_device(path, device: int | None = None, validate: bool = True, chunk: int = 1 << 26):
    """DeviceYearEventTable straight from an ARE1 file: ids + offsets to HBM,
    timestamps streamed through K0 (never kept).  Returns the table; its
    `violations()` holds the YET validation report."""
    from .resident import DeviceYearEventTable

    path = os.fspath(path)
    catalog, trials, total = _header(path)
    offsets, ids, ts = _maps(path, trials, total)
    dyet = DeviceYearEventTable.from_host_arrays(catalog, ids, np.array(offsets), device=device, chunk=chunk)
    if validate:
        dyet.validate_timestamps(ts, chunk=chunk)
    return dyet
