"""Multi-GPU group through the C ABI (8(e)).

worker_count > 1 runs the reference's trial ranges (split_by_events, the
partition rule of engine/__init__.py:151-159) on a GPU group in one library
call.  On a one-GPU box the group repeats device 0 (ARE_GROUP_DEVICES), so the
sharding, per-shard uploads, K0 report merge, the per-shard K2 launches, the
disjoint output ranges and the peer gather for K3 all run for real; with
several GPUs visible the last test uses every one of them.  The YLT must be
bitwise identical to the single-GPU run for any number of shards."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from paper_1308_2066_b200 import _native
from paper_1308_2066_b200.direct_access import TableSet
from paper_1308_2066_b200.engine import EngineConfig, price_layer, run_aggregate_analysis_with_stats
from paper_1308_2066_b200.errors import PortfolioInvalidError
from paper_1308_2066_b200.group import ShardedYearEventTable, shard_bounds, visible_devices
from paper_1308_2066_b200.portfolio import EventLossTable, Layer, LayerTerms, Trial, YearEventTable
from paper_1308_2066_b200.risk import order_stats
from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_yet

pytestmark = pytest.mark.gpu


def _portfolio(trials=3000, seed=7):
    spec = GeneratorSpec(seed=seed, catalog_size=20_000, trial_count=trials, events_per_trial_range=(1, 400),
                         elt_count=6, elt_size_range=(500, 3000))
    yet = generate_yet(spec)
    elts = tuple(generate_elt(spec, i) for i in range(6))
    layers = [Layer("a", elts[:4], LayerTerms(50.0, 2000.0, 3000.0, 40_000.0)),
              Layer("b", elts[2:], LayerTerms(0.0, float("inf"), 500.0, 25_000.0))]
    return layers, yet


@pytest.mark.parametrize("shards", [2, 3, 5])
@pytest.mark.parametrize("promote", [False, True])
def test_worker_count_group_is_bitwise_single_gpu(monkeypatch, shards, promote):
    import paper_1308_2066_b200.engine as engine

    layers, yet = _portfolio()
    want, ws = run_aggregate_analysis_with_stats(layers, yet, EngineConfig(worker_count=1))
    monkeypatch.setenv("ARE_GROUP_DEVICES", ",".join(["0"] * shards))
    if promote:  # the HBM-resident sharded YET (are_yet_upload + are_run_layer)
        monkeypatch.setattr(engine, "PROMOTE_MIN_OCC", 1)
    got, gs = run_aggregate_analysis_with_stats(layers, yet, EngineConfig(worker_count=shards))
    assert [y.losses.tobytes() for y in got] == [y.losses.tobytes() for y in want]
    assert (gs.trials, gs.layers, gs.lookups) == (ws.trials, ws.layers, ws.lookups)


def test_price_layer_on_group_matches(monkeypatch):
    layers, yet = _portfolio(trials=1234, seed=3)
    tset = TableSet.from_elts(layers[0].elts, yet.catalog_size)
    a, la = price_layer(yet, tset, [3, 0, 2], layers[0].terms)
    monkeypatch.setenv("ARE_GROUP_DEVICES", "0,0,0,0")
    b, lb = price_layer(yet, tset, [3, 0, 2], layers[0].terms, EngineConfig(worker_count=4))
    assert a.tobytes() == b.tobytes() and la == lb


def test_run_layer_c_abi_gathers_for_k3():
    """are_yet_upload -> are_run_layer(rps): the slices land in disjoint ranges
    of the caller's buffer and K3 on the gathered table gives the single-GPU
    order statistics."""
    layers, yet = _portfolio(trials=5000, seed=11)
    layer = layers[0]
    tset = TableSet.from_elts(layer.elts, yet.catalog_size)
    single, _ = price_layer(yet, tset, None, layer.terms)
    rps = [10.0, 50.0, 100.0, 250.0]
    pml_1, tvar_1 = order_stats(single, rps)
    syet = ShardedYearEventTable(yet, (0, 0, 0))
    assert syet.n_shards == 3 and list(syet.bounds) == list(shard_bounds(yet.offsets, 3))
    plans = [tset.plan(*tset.selection_arrays(None), device=0) for _ in range(3)]
    out = np.full(yet.trial_count, np.nan)
    lookups, pml, tvar = syet.run_layer(plans, layer.terms, out, rps=rps)
    assert out.tobytes() == single.tobytes()
    assert lookups == len(layer.elts) * int(yet.offsets[-1])
    assert list(pml) == list(pml_1)
    np.testing.assert_allclose(tvar, tvar_1, rtol=1e-12)
    # a sub-range writes only its own slots
    part = np.full(yet.trial_count, -1.0)
    syet.run_layer(plans, layer.terms, part, first=1000, last=4100)
    assert part[1000:4100].tobytes() == single[1000:4100].tobytes()
    assert np.all(part[:1000] == -1.0) and np.all(part[4100:] == -1.0)


def test_run_layer_gather_paths_agree():
    """With return periods the shards' K2 store each trial's loss straight
    into the table gathered on the first GPU (peer stores, fused gather);
    ARE_GROUP_NO_FUSE=1 runs the peer-copy gather instead.  Both must give
    the single-GPU YLT and order statistics (the check above, in a fresh
    process with the variable set)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, ARE_GROUP_NO_FUSE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "tests/test_gpu_group.py::test_run_layer_c_abi_gathers_for_k3"],
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_sharded_k0_report_equals_reference_fixture():
    """The merged per-shard K0 report reproduces the reference's
    validate_portfolio text (tests/golden/validation.json.gz)."""
    from paper_1308_2066_b200.portfolio import validate_portfolio
    from tests.validation_cases import build, load_cases

    n = 0
    for case in load_cases():
        layers, yet = build(case)
        if yet.offsets.size < 4:
            continue
        syet = ShardedYearEventTable(yet, (0, 0, 0))
        got = [str(v) for v in validate_portfolio(layers, syet)]
        assert got == case["report"], case["name"]
        n += 1
    assert n >= 40


def test_sharded_out_of_range_ids_are_refused(monkeypatch):
    import paper_1308_2066_b200.engine as engine

    layers, yet = _portfolio(trials=600)
    ids = yet.event_ids.copy()
    ids[int(yet.offsets[450]) + 1] = yet.catalog_size + 5  # in the last shard
    bad = YearEventTable(yet.catalog_size, ids, yet.timestamps, yet.offsets)
    monkeypatch.setenv("ARE_GROUP_DEVICES", "0,0")
    monkeypatch.setattr(engine, "PROMOTE_MIN_OCC", 1)
    with pytest.raises(PortfolioInvalidError) as err:
        engine.run_aggregate_analysis(layers, bad, EngineConfig(worker_count=2))
    assert "event_out_of_range" in {v.category for v in err.value.violations}


def test_every_visible_gpu():
    """The group over every GPU of the box (one on the single-GPU boxes)."""
    layers, yet = _portfolio(trials=2000, seed=5)
    n = visible_devices()
    want, _ = run_aggregate_analysis_with_stats(layers, yet, EngineConfig(worker_count=1))
    got, _ = run_aggregate_analysis_with_stats(layers, yet, EngineConfig(worker_count=max(n, 2)))
    assert [y.losses.tobytes() for y in got] == [y.losses.tobytes() for y in want]
    from paper_1308_2066_b200.group import devices_for

    assert devices_for(max(n, 2)) == tuple(range(n))
    if n > 1:
        size = _native._I32()
        _native.check(_native.load().are_group_size(ctypes.byref(size)))
        assert size.value == n


def test_group_calls_keep_the_callers_device():
    import torch

    torch.cuda.set_device(0)
    ShardedYearEventTable(_portfolio(trials=100)[1], (0, 0))
    assert torch.cuda.current_device() == 0
