"""Host -> HBM streaming for large host arrays (YET ids, timestamps).

A pageable numpy array (or a memmap) copies to the GPU at ~10 GB/s.  This
stages it through two pinned buffers: host threads fill buffer b (numpy's
copy releases the GIL) while the copy engine drains buffer 1-b, so the
transfer runs near the PCIe link rate.  Torch provides the pinned memory,
streams and events (plumbing); nothing here computes.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np


class Uploader:
    def __init__(self, chunk_bytes: int = 64 << 20, threads: int = 8):
        import torch

        self.torch = torch
        self.chunk_bytes = chunk_bytes
        self.bufs = [torch.empty(chunk_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.events = [torch.cuda.Event() for _ in range(2)]
        self.stream = torch.cuda.Stream()
        self.pool = ThreadPoolExecutor(max_workers=max(1, threads))
        self.threads = max(1, threads)

    def _fill(self, dst: np.ndarray, src: np.ndarray) -> None:
        n = src.shape[0]
        step = (n + self.threads - 1) // self.threads
        parts = [(a, min(n, a + step)) for a in range(0, n, step)]
        list(self.pool.map(lambda ab: np.copyto(dst[ab[0]:ab[1]], src[ab[0]:ab[1]]), parts))

    def copy(self, dst_tensor, src: np.ndarray) -> None:
        """dst_tensor[:len(src)] <- src (byte-identical; dtype sizes must match)."""
        torch = self.torch
        src = np.asarray(src)
        flat = dst_tensor.view(torch.uint8)
        nbytes = src.nbytes
        raw = src.reshape(-1).view(np.uint8) if src.flags.c_contiguous else np.ascontiguousarray(src).view(np.uint8)
        # the destination may have been written (e.g. zero-filled) on the
        # caller's stream: the copies must land after that work
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            for i, a in enumerate(range(0, nbytes, self.chunk_bytes)):
                b = min(nbytes, a + self.chunk_bytes)
                k = i & 1
                self.events[k].synchronize()  # buffer k drained by its previous copy
                host = self.bufs[k].numpy()
                self._fill(host[: b - a], raw[a:b])
                flat[a:b].copy_(self.bufs[k][: b - a], non_blocking=True)
                self.events[k].record(self.stream)
        self.stream.synchronize()

    def close(self) -> None:
        self.pool.shutdown(wait=False)
