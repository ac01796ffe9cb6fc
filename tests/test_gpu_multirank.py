"""Two ranks, one GPU: the bench's N>1 path with the real K2.

Two processes share cuda:0 over gloo (NCCL refuses two ranks on one GPU).  Each
rank uploads only its `partition(offsets, 2)` shard of the YET -- the trial
range split_by_events gives it (reference engine/__init__.py:151-159) -- runs
K2 on it, and the exchange functions reassemble the full YLT (allgather_ylt)
and the C3 block (allgather_portfolio: per-rank roll-up, then one gather).
Everything gathered must be bitwise equal to a one-rank run over the whole
YET, and that run bitwise equal to the CPU oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_TERMS = [(500.0, 10_000.0, 20_000.0, 60_000.0), (250.0, 10_000.0, 0.0, float("inf")),
          (0.0, float("inf"), 30_000.0, 120_000.0)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _portfolio():
    from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet

    spec = GeneratorSpec(seed=1308, catalog_size=100_000, trial_count=6_001, events_per_trial_range=(1, 900),
                         elt_count=8, elt_size_range=(2_000, 8_000))
    return generate_yet(spec), tuple(generate_elt(spec, i) for i in range(spec.elt_count)), spec.catalog_size


def _shard(yet, a: int, b: int):
    from paper_1308_2066_b200.portfolio import YearEventTable

    lo, hi = int(yet.offsets[a]), int(yet.offsets[b])
    return YearEventTable(yet.catalog_size, yet.event_ids[lo:hi], None, yet.offsets[a:b + 1] - lo)


def _run(yet, elts, catalog):
    """K2 for every layer of _TERMS over `yet` on cuda:0: (L, T) float64 on the device."""
    import torch

    from paper_1308_2066_b200.direct_access import TableSet
    from paper_1308_2066_b200.portfolio import LayerTerms
    from paper_1308_2066_b200.resident import DeviceYearEventTable

    tset = TableSet.from_elts(elts, catalog)
    plan = tset.plan(*tset.selection_arrays(None))
    dyet = DeviceYearEventTable.from_host_arrays(catalog, yet.event_ids, yet.offsets, device=0)
    out = torch.empty((len(_TERMS), dyet.trial_count), dtype=torch.float64, device="cuda:0")
    for i, t in enumerate(_TERMS):
        dyet.simulate_device(plan, LayerTerms(*t), out=out[i])
    torch.cuda.synchronize()
    return out


def _rank(rank: int, world: int, port: int, q) -> None:
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1308_2066_b200.distributed import allgather_portfolio, allgather_ylt, partition

        yet, elts, catalog = _portfolio()
        parts = partition(yet.offsets, world)
        a, b = parts[rank]
        local = _run(_shard(yet, a, b), elts, catalog).cpu()
        full = allgather_ylt(local[0].contiguous(), parts)
        rows, port_ylt = allgather_portfolio([local[i].contiguous() for i in range(len(_TERMS))], parts)
        q.put((rank, parts, full.numpy().tobytes(), [r.numpy().tobytes() for r in rows], port_ylt.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_cuda0_bitwise_one_rank():
    import torch
    import torch.multiprocessing as mp

    import oracle

    yet, elts, catalog = _portfolio()
    single = _run(yet, elts, catalog).cpu().numpy()
    # the one-rank run itself is pinned to the oracle (first layer, first 600 trials)
    stacked = oracle.dense_tables(elts, catalog)
    fin = [np.array([getattr(e.terms, f) for e in elts]) for f in
           ("exchange_rate", "event_retention", "event_limit", "share")]
    want = np.zeros(yet.trial_count)
    oracle.run_trials_port(yet.event_ids, yet.offsets, stacked, np.arange(len(elts), dtype=np.int64), *fin,
                           *_TERMS[0], 0, 0, 600, want)
    assert single[0, :600].tobytes() == want[:600].tobytes()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    port_want = single[0].copy()
    for i in range(1, len(_TERMS)):
        port_want = port_want + single[i]
    for rank, parts, full, rows, port_ylt in got:
        assert len(parts) == 2 and parts[0][0] == 0 and parts[1][1] == yet.trial_count
        assert 0 < parts[0][1] == parts[1][0] < yet.trial_count, "both ranks own trials"
        assert full == single[0].tobytes(), f"rank {rank}: gathered YLT differs from the one-rank run"
        for i, r in enumerate(rows):
            assert r == single[i].tobytes(), f"rank {rank}: layer {i} differs"
        assert port_ylt == port_want.tobytes(), f"rank {rank}: portfolio roll-up differs"
    assert torch.cuda.is_available()
