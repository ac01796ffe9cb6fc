"""Multi-GPU sharding of the trial dimension (one process per GPU).

Trials are independent and every YLT slot is written by exactly one trial
(SPEC.md:276), so the simulation shards with no data-path collective:
rank r simulates the contiguous, occurrence-balanced trial range
`partition(offsets, world)[r]` -- the reference's own `_split_by_events`
rule (engine/__init__.py:151-159) with parts = world size -- against its own
replica of the tables.  The one real exchange is the YLT gather that the
global PML/TVaR order statistics need: a single all-gather of the float64
slices over NCCL (NVLink/NVSwitch on a B200 node), after which every rank
holds the full YLT and runs K3 on it.  The YLT is bit-identical for any
world size because each trial's value does not depend on the partition.

The same functions run over gloo on CPU tensors, which is how
tests/test_distributed.py covers the N>1 logic without GPUs.
"""

from __future__ import annotations

import numpy as np

from .engine import split_by_events


def partition(offsets: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Trial range per rank; ranks beyond the available batches get (n, n)."""
    n = int(offsets.shape[0]) - 1
    parts = split_by_events(offsets, world) if n > 0 else []
    parts = parts + [(n, n)] * (world - len(parts))
    return parts


def allgather_ylt(local, parts: list[tuple[int, int]], group=None):
    """Concatenate every rank's YLT slice (in partition order) on every rank."""
    import torch
    import torch.distributed as dist

    world = len(parts)
    width = max(b - a for a, b in parts) if parts else 0
    pad = torch.zeros(max(width, 1), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = torch.empty(world * max(width, 1), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(bufs, pad, group=group)
    chunks = [bufs[r * max(width, 1): r * max(width, 1) + (b - a)] for r, (a, b) in enumerate(parts)]
    return torch.cat(chunks)


def allgather_portfolio(local_layers, parts: list[tuple[int, int]], group=None):
    """The C3 exchange: this rank first rolls its L layer
    slices up into its portfolio slice -- the roll-up is per trial
    (metrics.py:118-133), so it commutes with the trial sharding -- then ONE
    all-gather moves the (L + 1)-row block.  Returns (the L full layer YLTs,
    the full portfolio YLT), every one bit-identical to a single-GPU run."""
    import torch
    import torch.distributed as dist

    layers = list(local_layers)
    if not layers:
        raise ValueError("no layer slices to gather")
    n_layers, n = len(layers), int(layers[0].shape[0])
    if n_layers == 1:
        port = layers[0].clone()
    elif layers[0].is_cuda:
        from .risk import rollup_device

        port = rollup_device(layers)
    else:  # CPU tensors (gloo): the same left-to-right float64 sum
        port = layers[0].clone()
        for y in layers[1:]:
            port = port + y
    world = len(parts)
    width = max(1, max(b - a for a, b in parts))
    block = torch.zeros((n_layers + 1, width), dtype=torch.float64, device=layers[0].device)
    if n:
        block[:n_layers, :n] = torch.stack(layers)
        block[n_layers, :n] = port
    bufs = torch.empty((world, n_layers + 1, width), dtype=torch.float64, device=block.device)
    dist.all_gather_into_tensor(bufs.view(-1), block.view(-1), group=group)
    rows = [torch.cat([bufs[r, row, : b - a] for r, (a, b) in enumerate(parts)]) for row in range(n_layers + 1)]
    return rows[:n_layers], rows[n_layers]


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a host scalar over ranks (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
