"""HBM-resident year event tables and year loss tables.

`DeviceYearEventTable` uploads a YET's uint32 ids and int64 offsets to the
GPU once (timestamps are never read by the simulation) so that
repeated pricing -- the paper's interactive re-pricing scenario and the
reference's session reprice (service.py:213-241 -> price_layer) -- streams
only HBM, never PCIe.  Device memory and streams come from torch (plumbing);
the compute is K2 in libaggrisk_b200.so.

It is accepted by `price_layer` / `run_aggregate_analysis` in place of a host
`YearEventTable` (same `catalog_size`, `offsets`, `trial_count`), and its
`simulate_device` returns the YLT as a CUDA tensor for `risk.order_stats`.
"""

from __future__ import annotations

import ctypes
import os
import warnings

import numpy as np

from . import _native
from .portfolio import MAX_TRIAL_LENGTH


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 engine has no CPU fallback")
    return torch


_UPLOADERS: dict = {}


def _uploader(device):
    """The host->device staging pipeline of `device` (its own stream, events
    and pinned buffers, created under that device: a copy to another GPU never
    runs on the first GPU's stream)."""
    torch = _torch()
    idx = torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    up = _UPLOADERS.get(idx)
    if up is None:
        from .h2d import Uploader

        import os

        with torch.cuda.device(idx):
            # the staging copies are host-memory bound: use the cores we have
            up = Uploader(threads=max(1, min(16, len(os.sched_getaffinity(0)))))
        _UPLOADERS[idx] = up
    return up


class _Resident:
    def __init__(self, owner: "DeviceYearEventTable"):
        self.owner = owner

    def simulate(self, plan, n_sel, terms, out: np.ndarray, variant: str) -> int:
        d_out = self.owner.simulate_device(plan, terms, variant=variant)
        out[:] = d_out.cpu().numpy()
        return int(n_sel) * int(self.owner.offsets[-1])


class DeviceYearEventTable:
    """A YET whose ids/offsets live in HBM (validated on the device, K0)."""

    def __init__(self, yet, device: int | None = None, host_yet=None):
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._upload(yet.catalog_size, yet.event_ids, yet.offsets, dev)
        self.host = host_yet if host_yet is not None else yet
        ts = getattr(yet, "timestamps", None)
        if ts is not None:
            self.validate_timestamps(ts)

    @classmethod
    def from_host_arrays(cls, catalog_size: int, ids, offsets, device: int | None = None, chunk: int = 1 << 26):
        """Upload ids (any uint32 array-like, e.g. a memmap) in `chunk`-id pieces."""
        torch = _torch()
        self = cls.__new__(cls)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._upload(catalog_size, ids, offsets, dev, chunk)
        self.host = None
        return self

    @classmethod
    def from_device(cls, catalog_size: int, d_ids, d_offsets, host_offsets: np.ndarray):
        """Wrap tensors already in HBM (int32-viewed uint32 ids, int64 offsets)."""
        self = cls.__new__(cls)
        self.device = d_ids.device
        self.catalog_size = int(catalog_size)
        self.offsets = np.ascontiguousarray(host_offsets, dtype=np.int64)
        self.host = None
        self.d_ids, self.d_offsets = d_ids, d_offsets
        self._n_ids = int(d_ids.numel())
        self._report = None
        self._validate_ids()
        self._device = _Resident(self)
        return self

    def _upload(self, catalog_size, ids, offsets, dev, chunk: int = 1 << 26) -> None:
        torch = _torch()
        self.device = dev
        self.catalog_size = int(catalog_size)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        n = int(self.offsets[-1])
        # +4 zero ids of padding: 16-byte loads past the last trial stay in
        # bounds (only the padding is zeroed; the upload overwrites the rest)
        self.d_ids = torch.empty(n + 4, dtype=torch.int32, device=dev)
        self.d_ids[n:].zero_()
        if n:
            src = ids if getattr(ids, "dtype", None) == np.uint32 else np.asarray(ids, dtype=np.uint32)
            with torch.cuda.device(dev):
                _uploader(dev).copy(self.d_ids[:n], src)
        self._n_ids = n
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)  # read-only numpy source
            self.d_offsets = torch.from_numpy(self.offsets).to(dev)
        self._report = None
        self._validate_ids()
        self._device = _Resident(self)

    # ---- K0 validation ------------------------------------------------------
    def _k0(self, d_ts=None, ts_base: int = 0, t0: int = 0, t1: int | None = None, ids: bool = True):
        torch = _torch()
        t1 = self.trial_count if t1 is None else t1
        rep = _native.YetReport()
        st = torch.cuda.current_stream(self.device)
        _native.check(_native.load().are_validate_yet_device(
            self.d_ids.data_ptr(), self._n_ids if ids else 0, self.d_offsets.data_ptr() + 8 * t0, t1 - t0, t0,
            None if d_ts is None else d_ts.data_ptr(), ts_base, MAX_TRIAL_LENGTH, ctypes.byref(rep),
            ctypes.c_void_p(st.cuda_stream)))
        return rep

    def _validate_ids(self) -> None:
        """Ids range + trial lengths, one device pass at upload.  Every later
        K2 launch over this table then skips its per-id range check."""
        rep = self._k0()
        self._report = {"min_id": int(rep.min_id), "max_id": int(rep.max_id), "bad_trials": int(rep.bad_trials),
                        "first_bad": int(rep.first_bad_trial), "unsorted": 0, "ts_nan": 0,
                        "ts_min": None, "ts_max": None}
        self.ids_validated = self._n_ids == 0 or rep.max_id <= self.catalog_size
        self._pack_ids()

    def _pack_ids(self) -> None:
        """The packed resident id layout (are_yet_pack_device: three 21-bit
        ids per 64-bit word, 2/3 of the uint32 bytes) that the relay kernel
        streams instead of the uint32 ids.  Built once, beside the uint32
        ids, for validated tables whose ids fit 21 bits, when ARE_PACKED_IDS=1
        (opt-in: 1.79 vs 1.82 ms per C2 K2 launch, for 2/3 more id memory;
        DESIGN.md section 4)."""
        self.d_packed = None
        if not (self.ids_validated and self._n_ids and int(self._report["max_id"]) < (1 << 21)):
            return
        if os.environ.get("ARE_PACKED_IDS", "0") != "1":
            return
        torch = _torch()
        lib = _native.load()
        words = int(lib.are_packed_id_words(self._n_ids))
        d_packed = torch.empty(words, dtype=torch.int64, device=self.device)
        st = torch.cuda.current_stream(self.device)
        _native.check(lib.are_yet_pack_device(self.device.index, self.d_ids.data_ptr(), self._n_ids,
                                              d_packed.data_ptr(), None, ctypes.c_void_p(st.cuda_stream)))
        self.d_packed = d_packed

    def ids_flag(self, plan) -> int:
        """IDS_VALIDATED when every id of this table indexes inside the plan's
        rows (max id < row_len): a plan over a smaller catalog than the YET's
        keeps K2's per-id range check."""
        if not self.ids_validated:
            return 0
        if self._n_ids and _native.plan_info(plan).row_len <= int(self._report["max_id"]):
            return 0
        return _native.IDS_VALIDATED

    def validate_timestamps(self, ts, chunk: int = 1 << 26) -> None:
        """Stream host timestamps through K0 in trial-aligned chunks (kept nowhere)."""
        torch = _torch()
        n_trials = self.trial_count
        r = self._report
        t0 = 0
        while t0 < n_trials:
            a = int(self.offsets[t0])
            t1 = int(np.searchsorted(self.offsets, a + chunk, side="right")) - 1
            t1 = min(max(t1, t0 + 1), n_trials)
            b = int(self.offsets[t1])
            d_ts = torch.empty(max(b - a, 1), dtype=torch.float64, device=self.device)
            if b > a:
                with torch.cuda.device(self.device):
                    _uploader(self.device).copy(d_ts, np.asarray(ts[a:b], dtype=np.float64))
            rep = self._k0(d_ts, ts_base=a, t0=t0, t1=t1, ids=False)
            r["unsorted"] += int(rep.unsorted)
            r["ts_nan"] += int(rep.ts_nan)
            if b > a and rep.ts_nan < (b - a):
                r["ts_min"] = rep.ts_min if r["ts_min"] is None else min(r["ts_min"], rep.ts_min)
                r["ts_max"] = rep.ts_max if r["ts_max"] is None else max(r["ts_max"], rep.ts_max)
            t0 = t1
        r["ts_checked"] = True

    def yet_violations(self):
        """The YET half of validate_portfolio (model.py:371-395) from K0's counters."""
        from .portfolio import Violation

        r = self._report
        out = []
        if self.trial_count == 0:
            out.append(Violation("no_trials", "year event table holds no trials"))
        if r["bad_trials"]:
            out.append(Violation("trial_length", f"{r['bad_trials']} trial(s) outside [1, {MAX_TRIAL_LENGTH}] "
                                                 f"occurrences (first: trial {r['first_bad']})"))
        if self._n_ids:
            if r["min_id"] < 1 or r["max_id"] > self.catalog_size:
                out.append(Violation("event_out_of_range", f"trial event id outside [1, {self.catalog_size}]"))
            # numpy's min/max propagate NaN, and a NaN compares false: no violation
            if r.get("ts_checked") and not r["ts_nan"] and r["ts_min"] is not None and \
                    (r["ts_min"] < 0.0 or r["ts_max"] > 1.0):
                out.append(Violation("bad_timestamp", "timestamps must lie in [0, 1]"))
            if r["unsorted"]:
                out.append(Violation("trial_unsorted", f"timestamps decrease inside {r['unsorted']} position(s)"))
        return out

    @property
    def trial_count(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def event_ids(self) -> np.ndarray:  # host view for validation
        if self.host is None:
            raise AttributeError("device-only YET has no host event ids")
        return self.host.event_ids

    @property
    def timestamps(self):
        return None if self.host is None else getattr(self.host, "timestamps", None)

    def simulate_device(self, plan, terms, first: int = 0, last: int | None = None, out=None,
                        stream=None, variant: str = "auto", check: bool = True, flags: int = 0):
        """K2 over trials [first, last) into a float64 CUDA tensor (allocated
        when `out` is None); launches on `stream` (default: torch's current)."""
        torch = _torch()
        n = self.trial_count
        last = n if last is None else last
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=self.device)
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        lib = _native.load()
        flag = self.ids_flag(plan)
        args = (self._n_ids, self.d_offsets.data_ptr(), n,
                int(first), int(last), float(terms.occ_retention), float(terms.occ_limit),
                float(terms.agg_retention), float(terms.agg_limit), out.data_ptr(),
                ctypes.c_void_p(st.cuda_stream), _native.VARIANTS[variant] | flag | int(flags))
        if self.d_packed is not None and flag:
            _native.check(lib.are_simulate_device_packed(plan.value, self.d_ids.data_ptr(),
                                                         self.d_packed.data_ptr(), *args))
        else:
            _native.check(lib.are_simulate_device(plan.value, self.d_ids.data_ptr(), *args))
        if check and not flag:  # validated ids cannot raise the range flag
            _native.check(lib.are_check_errors(plan.value, ctypes.c_void_p(st.cuda_stream)))
        return out
