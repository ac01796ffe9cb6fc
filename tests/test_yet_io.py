"""ARE1 binary YET I/O (host side, no GPU): the reference-written fixture
loads bit-exactly, save/load round-trips, and the reference's error classes
fire for damaged files (pkg/src/aggrisk/io.py:63-201)."""

from __future__ import annotations

import hashlib
import os
import struct

import numpy as np
import pytest

from paper_1308_2066_b200.errors import (
    DataFormatError,
    FormatMismatchError,
    TruncatedPayloadError,
    VersionMismatchError,
)
from paper_1308_2066_b200.yet_io import load_yet, save_yet
from tests.conftest import GOLDEN

FIXTURE = os.path.join(GOLDEN, "yet_small.are1")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_reference_written_file_loads_bit_exact(golden):
    g = golden["are1"]
    yet = load_yet(FIXTURE)
    assert yet.catalog_size == g["catalog"] and yet.trial_count == g["trials"]
    assert sha(yet.event_ids) == g["ids_sha256"]
    assert sha(yet.offsets) == g["offsets_sha256"]
    assert sha(yet.timestamps) == g["timestamps_sha256"]
    ids_only = load_yet(FIXTURE, ids_only=True)
    assert ids_only.timestamps is None and sha(ids_only.event_ids) == g["ids_sha256"]


def test_save_reproduces_reference_bytes(tmp_path):
    yet = load_yet(FIXTURE)
    out = tmp_path / "copy.are1"
    save_yet(yet, out)
    assert out.read_bytes() == open(FIXTURE, "rb").read()


def _damaged(tmp_path, mutate) -> str:
    raw = bytearray(open(FIXTURE, "rb").read())
    raw = mutate(raw)
    p = tmp_path / "bad.are1"
    p.write_bytes(bytes(raw))
    return str(p)


@pytest.mark.parametrize("mutate,err", [
    (lambda r: b"XXXX" + r[4:], FormatMismatchError),
    (lambda r: r[:4] + struct.pack("<HH", 2, 1) + r[8:], VersionMismatchError),
    (lambda r: r[:4] + struct.pack("<HH", 1, 9) + r[8:], FormatMismatchError),
    (lambda r: r[:4] + struct.pack("<HH", 1, 2) + r[8:], FormatMismatchError),
    (lambda r: r[:-5], TruncatedPayloadError),
    (lambda r: r[:20], TruncatedPayloadError),
    (lambda r: r + b"\0\0", DataFormatError),
])
def test_damaged_files_raise_reference_errors(tmp_path, mutate, err):
    with pytest.raises(err):
        load_yet(_damaged(tmp_path, mutate))
