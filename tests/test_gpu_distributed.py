"""The N>1 exchange functions on the GPU path: a one-rank NCCL group (the
GPU box has one B200) running allgather_ylt and allgather_portfolio on CUDA
tensors, the portfolio roll-up through the device kernel (k3_rollup)."""

from __future__ import annotations

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_one_rank_exchange(rng):
    import torch
    import torch.distributed as dist

    from paper_1308_2066_b200.distributed import allgather_portfolio, allgather_ylt, partition

    store = dist.TCPStore("127.0.0.1", _free_port(), 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 100_003
        offsets = np.arange(n + 1, dtype=np.int64) * 7
        parts = partition(offsets, 1)
        assert parts == [(0, n)]
        layers = [torch.from_numpy(rng.random(n) * 1e4).cuda() for _ in range(5)]
        full = allgather_ylt(layers[0], parts)
        assert torch.equal(full, layers[0])
        got_layers, port = allgather_portfolio(layers, parts)
        want = layers[0].cpu().numpy().copy()
        for y in layers[1:]:
            want = want + y.cpu().numpy()
        assert all(torch.equal(g, w) for g, w in zip(got_layers, layers))
        assert port.cpu().numpy().tobytes() == want.tobytes()
    finally:
        dist.destroy_process_group()
