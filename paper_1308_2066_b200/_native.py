"""ctypes binding of ``libaggrisk_b200.so`` (declared in ``include/aggrisk_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1308_2066_b200/csrc``).  There is no CPU fallback: if the
library is missing or no B200 is visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import EventOutOfRangeError

# ARE_LIB overrides the library path (kernel A/B experiments with alternative builds)
LIB_PATH = os.environ.get("ARE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     "libaggrisk_b200.so")

ARE_OK, ARE_EINVAL, ARE_ERANGE, ARE_ECUDA, ARE_ENOMEM, ARE_EINDEX = range(6)
VARIANTS = {"auto": 0, "hotset": 1, "dense": 2}
IDS_VALIDATED = 0x100  # ARE_FLAG_IDS_VALIDATED: every YET id is known to be <= catalog
def spare_sms(k: int) -> int:
    """ARE_SPARE_SMS(k): K2 leaves k SMs to concurrent work on another stream."""
    return (int(k) & 0xFF) << 12

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double


class YetReport(ctypes.Structure):
    _fields_ = [
        ("min_id", ctypes.c_uint32),
        ("max_id", ctypes.c_uint32),
        ("bad_trials", _I64),
        ("first_bad_trial", _I64),
        ("unsorted", _I64),
        ("ts_nan", _I64),
        ("ts_min", _D),
        ("ts_max", _D),
        ("ts_checked", _I32),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_sel", _I64),
        ("row_len", _I64),
        ("hot_events", _I64),
        ("entries", _I64),
        ("overflow_entries", _I64),
        ("filter_bits", _I64),
        ("device_bytes", _I64),
        ("zero_skip_exact", _I32),
        ("smem_bytes", _I32),
        ("relay_filter_bits", _I64),
        ("relay", _I32),
        ("relay_smem_bytes", _I32),
    ]


# name -> (restype, argtypes); must match include/aggrisk_b200.h
SIGNATURES = {
    "are_last_error": (ctypes.c_char_p, []),
    "are_version": (ctypes.c_int, []),
    "are_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "are_select_device": (ctypes.c_int, [ctypes.c_int]),
    "are_device_sm_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "are_launch_count": (_I64, []),
    "are_host_register": (ctypes.c_int, [_P, _I64]),
    "are_host_unregister": (ctypes.c_int, [_P]),
    "are_host_is_pinned": (ctypes.c_int, [_P]),
    "are_tables_from_dense": (ctypes.c_int, [_P, _I64, _I64, ctypes.POINTER(_P)]),
    "are_tables_from_records": (ctypes.c_int, [_P, _P, _P, _I64, _I64, ctypes.POINTER(_P)]),
    "are_tables_info": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "are_tables_read_row": (ctypes.c_int, [_P, _I64, _P]),
    "are_tables_free": (ctypes.c_int, [_P]),
    "are_plan_build": (ctypes.c_int, [_P, _P, _I64, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "are_plan_build_pool": (ctypes.c_int, [_P, _P, _I64, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "are_plan_build_precombined": (ctypes.c_int, [_P, _P, _I64, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "are_plan_info": (ctypes.c_int, [_P, ctypes.POINTER(PlanInfo)]),
    "are_plan_free": (ctypes.c_int, [_P]),
    "are_simulate_device": (
        ctypes.c_int,
        [_P, _P, _I64, _P, _I64, _I64, _I64, _D, _D, _D, _D, _P, _P, _I32],
    ),
    "are_check_errors": (ctypes.c_int, [_P, _P]),
    "are_packed_id_words": (_I64, [_I64]),
    "are_yet_pack_device": (ctypes.c_int, [_I32, _P, _I64, _P, _P, _P]),
    "are_simulate_device_packed": (
        ctypes.c_int,
        [_P, _P, _P, _I64, _P, _I64, _I64, _I64, _D, _D, _D, _D, _P, _P, _I32],
    ),
    "are_simulate_layers_device": (
        ctypes.c_int, [_P, _I32, _P, _P, _P, _I64, _P, _I64, _I64, _I64, _P, _I64, _P, _I32]),
    "are_layer_table_build": (ctypes.c_int, [_P, _I32, _P, _P, _P, ctypes.POINTER(_P)]),
    "are_layer_table_free": (ctypes.c_int, [_P]),
    "are_simulate_layers_precombined": (
        ctypes.c_int, [_P, _P, _I64, _P, _I64, _I64, _I64, _P, _I64, _P, _I32]),
    "are_simulate_host": (
        ctypes.c_int,
        [_P, _P, _I64, _P, _I64, _I64, _I64, _D, _D, _D, _D, _P, ctypes.POINTER(_I64), _I32],
    ),
    "are_run_trials": (
        ctypes.c_int,
        [_P, _I64, _P, _I64, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P,
         _D, _D, _D, _D, _I64, _I64, _I64, _P, _I64, ctypes.POINTER(_I64)],
    ),
    "are_validate_yet_device": (
        ctypes.c_int, [_P, _I64, _P, _I64, _I64, _P, _I64, _I64, ctypes.POINTER(YetReport), _P]),
    "are_order_stats_device": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P, _P]),
    "are_order_stats_async": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _I32, _P]),
    "are_order_stats_host": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P]),
    "are_order_stats_summary_device": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P, _P, _P]),
    "are_pml_many_device": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P]),
    "are_rollup_device": (ctypes.c_int, [_P, _I64, _I64, _P, _P]),
    # multi-GPU group (capi_group.cu)
    "are_init": (ctypes.c_int, [ctypes.c_int]),
    "are_init_devices": (ctypes.c_int, [_P, _I32]),
    "are_shutdown": (ctypes.c_int, []),
    "are_group_size": (ctypes.c_int, [ctypes.POINTER(_I32)]),
    "are_group_device": (ctypes.c_int, [_I32, ctypes.POINTER(ctypes.c_int)]),
    "are_tables_device": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
    "are_plan_device": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
    "are_tables_replicate": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_P)]),
    "are_yet_upload": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P, _I32, _I64, ctypes.POINTER(_P)]),
    "are_yet_report": (ctypes.c_int, [_P, ctypes.POINTER(YetReport)]),
    "are_yet_shards": (ctypes.c_int, [_P, ctypes.POINTER(_I32), _P, _P]),
    "are_yet_free": (ctypes.c_int, [_P]),
    "are_run_layer": (ctypes.c_int, [_P, _P, _I32, _D, _D, _D, _D, _I64, _I64, _P, ctypes.POINTER(_I64), _I32,
                                     _P, _I64, _P, _P]),
    "are_run_layer_host": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _I32, _P, _D, _D, _D, _D, _I64, _I64, _P,
                                          ctypes.POINTER(_I64), _I32]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load the library once; raise ImportError when it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: the B200 engine has no CPU fallback; "
                    "build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().are_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Translate a status code into the reference's exception types."""
    if rc == ARE_OK:
        return
    msg = last_error()
    if rc == ARE_EINVAL:
        raise ValueError(msg)
    if rc == ARE_ERANGE:
        raise EventOutOfRangeError(msg)
    if rc == ARE_EINDEX:
        raise IndexError(msg)
    if rc == ARE_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"B200 engine: {msg}")


def ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


def launch_count() -> int:
    return int(load().are_launch_count())


class Handle:
    """Owns one native handle; frees it exactly once."""

    __slots__ = ("value", "_free", "__weakref__")

    def __init__(self, value: int, free_name: str):
        self.value = value
        self._free = free_name

    def close(self) -> None:
        if self.value:
            v, self.value = self.value, None
            if _lib is not None:
                getattr(_lib, self._free)(v)

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:
            pass


def tables_from_dense(stacked: np.ndarray) -> Handle:
    lib = load()
    out = _P()
    a = np.ascontiguousarray(stacked, dtype=np.float64)
    check(lib.are_tables_from_dense(ptr(a), a.shape[0], a.shape[1], ctypes.byref(out)))
    return Handle(out.value, "are_tables_free")


def tables_from_records(ids: np.ndarray, losses: np.ndarray, table_offsets: np.ndarray, row_len: int) -> Handle:
    lib = load()
    out = _P()
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    losses = np.ascontiguousarray(losses, dtype=np.float64)
    table_offsets = np.ascontiguousarray(table_offsets, dtype=np.int64)
    check(lib.are_tables_from_records(ptr(ids), ptr(losses), ptr(table_offsets),
                                      table_offsets.shape[0] - 1, row_len, ctypes.byref(out)))
    return Handle(out.value, "are_tables_free")


def read_row(tables: Handle, row: int, row_len: int) -> np.ndarray:
    out = np.empty(row_len, dtype=np.float64)
    check(load().are_tables_read_row(tables.value, row, ptr(out)))
    return out


def plan_build(tables: Handle, rows, rate, ret, lim, share, pool: bool = False,
               precombine: bool = False) -> Handle:
    lib = load()
    arrs = [np.ascontiguousarray(rows, dtype=np.int64)] + [
        np.ascontiguousarray(x, dtype=np.float64) for x in (rate, ret, lim, share)
    ]
    out = _P()
    fn = lib.are_plan_build_pool if pool else (lib.are_plan_build_precombined if precombine else lib.are_plan_build)
    check(fn(tables.value, ptr(arrs[0]), arrs[0].shape[0], *(ptr(x) for x in arrs[1:]), ctypes.byref(out)))
    return Handle(out.value, "are_plan_free")


def tables_device(tables: Handle) -> int:
    d = ctypes.c_int(0)
    check(load().are_tables_device(tables.value, ctypes.byref(d)))
    return int(d.value)


def tables_replicate(tables: Handle, device: int) -> Handle:
    out = _P()
    check(load().are_tables_replicate(tables.value, int(device), ctypes.byref(out)))
    return Handle(out.value, "are_tables_free")


def plan_info(plan: Handle) -> PlanInfo:
    info = PlanInfo()
    check(load().are_plan_info(plan.value, ctypes.byref(info)))
    return info
