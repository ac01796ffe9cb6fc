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
import warnings

import numpy as np

from . import _native


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 engine has no CPU fallback")
    return torch


class _Resident:
    def __init__(self, owner: "DeviceYearEventTable"):
        self.owner = owner

    def simulate(self, plan, n_sel, terms, out: np.ndarray, variant: str) -> int:
        d_out = self.owner.simulate_device(plan, terms, variant=variant)
        out[:] = d_out.cpu().numpy()
        return int(n_sel) * int(self.owner.offsets[-1])


class DeviceYearEventTable:
    """A YET whose ids/offsets live in HBM."""

    def __init__(self, yet, device: int | None = None, host_yet=None):
        torch = _torch()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.catalog_size = int(yet.catalog_size)
        self.offsets = np.ascontiguousarray(yet.offsets, dtype=np.int64)
        self.host = host_yet if host_yet is not None else yet
        ids = np.ascontiguousarray(yet.event_ids, dtype=np.uint32)
        # int32 view of the uint32 ids (torch has no general uint32 math); the
        # host buffer is only read (copied to HBM), never written
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            self.d_ids = torch.from_numpy(ids.view(np.int32)).to(self.device)
        self.d_offsets = torch.from_numpy(self.offsets).to(self.device)
        self._check_ids()
        self._device = _Resident(self)

    def _check_ids(self) -> None:
        """One device pass at upload: are all ids inside [0, catalog]?  Then
        every later K2 launch over this table skips its per-id range check."""
        if self.d_ids.numel() == 0:
            self.ids_validated = True
            return
        lo, hi = int(self.d_ids.min()), int(self.d_ids.max())  # ids >= 2^31 view as negative
        self.ids_validated = lo >= 0 and hi <= self.catalog_size

    @classmethod
    def from_device(cls, catalog_size: int, d_ids, d_offsets, host_offsets: np.ndarray):
        """Wrap tensors already in HBM (int32-viewed uint32 ids, int64 offsets)."""
        self = cls.__new__(cls)
        self.device = d_ids.device
        self.catalog_size = int(catalog_size)
        self.offsets = np.ascontiguousarray(host_offsets, dtype=np.int64)
        self.host = None
        self.d_ids, self.d_offsets = d_ids, d_offsets
        self._check_ids()
        self._device = _Resident(self)
        return self

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
                        stream=None, variant: str = "auto", check: bool = True):
        """K2 over trials [first, last) into a float64 CUDA tensor (allocated
        when `out` is None); launches on `stream` (default: torch's current)."""
        torch = _torch()
        n = self.trial_count
        last = n if last is None else last
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=self.device)
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        lib = _native.load()
        _native.check(lib.are_simulate_device(
            plan.value, self.d_ids.data_ptr(), int(self.d_ids.numel()), self.d_offsets.data_ptr(), n,
            int(first), int(last), float(terms.occ_retention), float(terms.occ_limit),
            float(terms.agg_retention), float(terms.agg_limit), out.data_ptr(),
            ctypes.c_void_p(st.cuda_stream),
            _native.VARIANTS[variant] | (_native.IDS_VALIDATED if self.ids_validated else 0)))
        if check:
            _native.check(lib.are_check_errors(plan.value, ctypes.c_void_p(st.cuda_stream)))
        return out
