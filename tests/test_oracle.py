"""Pins the CPU oracle (oracle/) to the reference's own outputs.

Runs on CPU (no GPU needed).  The C restatement of the reference hot loop
must reproduce the reference engine bit-for-bit on the golden vectors written
by tests/golden/make_golden.py; the compiled reference kernel (oracle/_ref,
when built) must agree with both.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

import oracle
from tests.conftest import GOLDEN


def _run_port(inst, chunk=0):
    out = np.empty(inst.yet.trial_count)
    rows = np.arange(len(inst.layer.elts), dtype=np.int64)
    t = inst.layer.terms
    n = oracle.run_trials_port(inst.yet.event_ids, inst.yet.offsets, inst.stacked, rows, *inst.fin(),
                               t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit,
                               chunk, 0, inst.yet.trial_count, out, np.empty(max(chunk, 1)))
    return out, n


def test_port_matches_reference_on_1000_instances(instances):
    assert len(instances) == 1000
    for inst in instances:
        got, lookups = _run_port(inst)
        assert got.tobytes() == inst.ylt.tobytes()
        assert lookups == len(inst.layer.elts) * int(inst.yet.offsets[-1])
        # the reference's independent naive oracle agrees within 1e-9
        np.testing.assert_allclose(got, inst.ylt_naive, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("chunk", [1, 3, 7, 12])
def test_port_chunked_is_bitwise_fused(instances, chunk):
    for inst in instances[:150]:
        got, _ = _run_port(inst, chunk)
        assert got.tobytes() == inst.ylt.tobytes()


def test_port_term_kats(golden):
    assert oracle.financial_terms(30.0, 2.0, 10.0, 40.0, 0.5) == golden["kats"]["fin_terms_30_2_10_40_half"] == 20.0
    assert oracle.occurrence_terms(100.0, 10.0, 60.0) == 60.0
    assert oracle.occurrence_terms(50.0, 10.0, 60.0) == 40.0
    assert oracle.occurrence_terms(5.0, 10.0, 60.0) == 0.0


def test_port_worked_example(golden):
    # ELT {4: 100, 9: 50}, terms (10, 60, 0, 150), trial [4, 9, 4] -> 150
    stacked = np.zeros((1, 11))
    stacked[0, 4], stacked[0, 9] = 100.0, 50.0
    out = np.empty(1)
    oracle.run_trials_port(np.array([4, 9, 4], np.uint32), np.array([0, 3], np.int64), stacked,
                           np.array([0], np.int64), np.ones(1), np.zeros(1), np.full(1, np.inf), np.ones(1),
                           10.0, 60.0, 0.0, 150.0, 0, 0, 1, out)
    assert out[0] == golden["kats"]["worked_example"] == 150.0


def test_port_rejects_reference_bad_arguments(instances):
    inst = instances[0]
    out = np.empty(inst.yet.trial_count)
    with pytest.raises(ValueError):  # scratch < chunk (_kernel.pyx:51-52)
        oracle.run_trials_port(inst.yet.event_ids, inst.yet.offsets, inst.stacked,
                               np.zeros(1, np.int64), *(a[:1] for a in inst.fin()), 0.0, 1.0, 0.0, 1.0,
                               4, 0, 1, out, np.empty(2))


def test_reference_kernel_agrees_with_port(instances):
    mod = oracle.ref_kernel()
    if mod is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    for inst in instances[:300]:
        out = np.empty(inst.yet.trial_count)
        rows = np.arange(len(inst.layer.elts), dtype=np.int64)
        t = inst.layer.terms
        mod.run_trials(inst.yet.event_ids, inst.yet.offsets, inst.stacked, rows, *inst.fin(),
                       t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit, 0, 0,
                       inst.yet.trial_count, out, np.empty(1))
        assert out.tobytes() == inst.ylt.tobytes()


def test_threaded_driver_is_partition_invariant(instances):
    inst = max(instances, key=lambda i: i.yet.trial_count)
    t = inst.layer.terms
    terms = (t.occ_retention, t.occ_limit, t.agg_retention, t.agg_limit)
    one, n1 = oracle.run_layer_cpu(inst.yet.event_ids, inst.yet.offsets, inst.stacked, inst.fin(), terms, 1, "port")
    four, n4 = oracle.run_layer_cpu(inst.yet.event_ids, inst.yet.offsets, inst.stacked, inst.fin(), terms, 4, "port")
    assert one.tobytes() == four.tobytes() == inst.ylt.tobytes()
    assert n1 == n4


def test_metrics_oracle_matches_reference():
    z = np.load(os.path.join(GOLDEN, "metrics_1004.npz"))
    b = z["bounds"]
    for i in range(b.size - 1):
        x = z["losses"][b[i]:b[i + 1]]
        for j, rp in enumerate(z["rps"][i]):
            assert oracle.pml(x, rp) == z["pml"][i, j]
            assert oracle.tvar(x, rp) == z["tvar"][i, j]


def test_metrics_oracle_kats(golden):
    k = golden["kats"]
    ramp = np.arange(1, 1001, dtype=np.float64)
    assert oracle.pml(ramp, 100.0) == k["pml_ramp1000_rp100"] == 990.0
    assert oracle.tvar(ramp, 100.0) == k["tvar_ramp1000_rp100"] == 995.0
    assert [list(p) for p in oracle.ep_points(ramp, [2.0, 10.0, 100.0])] == k["ep_ramp1000"]


def test_c1_reference_ylt_fixture(golden):
    """The committed C1 YLT is the reference's (sha256 recorded at generation)."""
    ylt = np.load(os.path.join(GOLDEN, "c1_ylt.npy"))
    assert hashlib.sha256(ylt.tobytes()).hexdigest() == golden["c1"]["ylt_sha256"]
    assert oracle.pml(ylt, 100.0) == golden["c1"]["pml"][3]
