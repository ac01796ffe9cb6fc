"""N>1 host logic on CPU: world-size-2 gloo run of the sharded pipeline.

Each rank takes its `partition(offsets, world)` trial range, computes its YLT
slice (here with the CPU oracle standing in for K2, which needs a GPU), and
`allgather_ylt` reassembles the full YLT on every rank; it must equal the
single-process YLT bit for bit, and max_over_ranks must agree across ranks.
The C3 exchange (`allgather_portfolio`: per-rank roll-up, one gather of the
L + 1 rows) must give the single-process layer YLTs and portfolio sum.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_2066_b200.distributed import allgather_portfolio, allgather_ylt, max_over_ranks, partition


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_ylt(inst, a: int, b: int, terms=None) -> np.ndarray:
    import oracle

    out = np.zeros(inst.yet.trial_count)
    rows = np.arange(len(inst.layer.elts), dtype=np.int64)
    t = inst.layer.terms if terms is None else terms
    oracle.run_trials_port(inst.yet.event_ids, inst.yet.offsets, inst.stacked, rows, *inst.fin(),
                           t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit, 0, a, b, out)
    return out[a:b]


def _portfolio_terms(inst):
    from paper_1308_2066_b200.portfolio import LayerTerms

    t = inst.layer.terms
    return [t, LayerTerms(t.occ_retention * 0.5, t.occ_limit, 0.0, float("inf")),
            LayerTerms(0.0, float("inf"), t.agg_retention, t.agg_limit * 2.0)]


def _worker(rank: int, world: int, port: int, q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.instances import load_instances

        insts = sorted(load_instances(), key=lambda i: -i.yet.trial_count)[:3]
        for inst in insts:
            parts = partition(inst.yet.offsets, world)
            a, b = parts[rank]
            local = torch.from_numpy(_shard_ylt(inst, a, b))
            full = allgather_ylt(local, parts).numpy()
            q.put((rank, full.tobytes() == inst.ylt.tobytes(), a, b))
        # C3 exchange: per-rank roll-up, one gather of the (L + 1)-row block
        inst = insts[0]
        parts = partition(inst.yet.offsets, world)
        a, b = parts[rank]
        terms = _portfolio_terms(inst)
        local = [torch.from_numpy(_shard_ylt(inst, a, b, t)) for t in terms]
        layers, port = allgather_portfolio(local, parts)
        n = inst.yet.trial_count
        full = [_shard_ylt(inst, 0, n, t) for t in terms]
        want = full[0].copy()
        for y in full[1:]:
            want = want + y
        ok = all(g.numpy().tobytes() == w.tobytes() for g, w in zip(layers, full))
        q.put((rank, ok and port.numpy().tobytes() == want.tobytes(), -2, -2))
        q.put((rank, max_over_ranks(float(rank + 1)) == float(world), -1, -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_sharded_ylt_is_bitwise():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    results = [q.get(timeout=10) for _ in range(world * 5)]
    assert all(ok for _, ok, _, _ in results)
    spans = sorted({(a, b) for r, ok, a, b in results if a >= 0 and r == 0})
    assert spans  # rank 0 owned a non-trivial range


def test_partition_pads_short_worlds():
    offs = np.array([0, 5, 9], dtype=np.int64)
    assert partition(offs, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert partition(np.zeros(1, np.int64), 2) == [(0, 0), (0, 0)]
