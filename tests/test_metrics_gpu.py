"""K3 (device order statistics) against the reference metrics.

PML: exact (an order statistic).  TVaR: rel 1e-12 (the reference's own bound
against its full-sort oracle, test_metrics.py:44-52) -- the device sums the
tail in a fixed order with double-double accumulation; numpy sums the
partitioned tail pairwise.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from paper_1308_2066_b200.portfolio import YearLossTable
from paper_1308_2066_b200.risk import ep_curve, order_stats, pml, portfolio_rollup, tvar
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _ramp(n=1000):
    return YearLossTable("ramp", np.arange(1, n + 1, dtype=np.float64))


def test_kats(golden):
    k = golden["kats"]
    assert pml(_ramp(), 100.0) == k["pml_ramp1000_rp100"] == 990.0
    assert tvar(_ramp(), 100.0) == k["tvar_ramp1000_rp100"] == 995.0
    c = ep_curve(_ramp(), [100.0, 2.0, 10.0, 2.0])
    assert [list(p) for p in c.points] == k["ep_ramp1000"]
    assert c.probabilities == (0.5, 0.1, 0.01)
    assert pml(_ramp(10), 10.0) == 9.0 and tvar(_ramp(10), 10.0) == 9.5
    assert pml(np.arange(10.0, 110.0, 10.0), 3.0) == k["pml_10_110_rp3"] == 70.0
    flat = YearLossTable("f", np.full(100, 7.5))
    assert pml(flat, 4.0) == 7.5 and tvar(flat, 4.0) == 7.5


def test_argument_errors():
    with pytest.raises(ValueError):
        pml(_ramp(100), 1.0)
    with pytest.raises(ValueError):
        pml(_ramp(100), 101.0)
    with pytest.raises(ValueError):
        pml(np.zeros(0), 2.0)
    with pytest.raises(ValueError):
        ep_curve(_ramp(), [])


def test_golden_random_ylts():
    z = np.load(os.path.join(GOLDEN, "metrics_1004.npz"))
    b = z["bounds"]
    for i in range(b.size - 1):
        x = z["losses"][b[i]:b[i + 1]]
        p, t = order_stats(x, z["rps"][i])
        assert list(p) == list(z["pml"][i])
        np.testing.assert_allclose(t, z["tvar"][i], rtol=1e-12)
        assert np.all(t >= p)


def test_large_ylt_with_ties_and_device_input(rng):
    import torch

    n = 1_000_000
    x = rng.lognormal(8.0, 1.5, n)
    x[rng.random(n) < 0.1] = 0.0
    x[rng.random(n) < 0.1] = 66_000.0  # agg-limit saturation ties, as in C1
    rps = [1.5, 2.0, 10.0, 50.0, 100.0, 250.0, 1000.0, 10_000.0, float(n)]
    p, t = order_stats(x, rps)
    for r, pv, tv in zip(rps, p, t):
        assert pv == oracle.pml(x, r)
        assert tv == pytest.approx(oracle.tvar(x, r), rel=1e-12)
    dp, dt = order_stats(torch.from_numpy(x).cuda(), rps)
    assert dp.tobytes() == p.tobytes() and dt.tobytes() == t.tobytes()  # deterministic


def test_rollup_bitwise(rng):
    ylts = [YearLossTable(str(i), rng.random(100_003) * 100.0) for i in range(70)]
    want = ylts[0].losses.copy()
    for y in ylts[1:]:
        np.add(want, y.losses, out=want)
    got = portfolio_rollup(ylts)
    assert got.layer_id == "portfolio" and got.losses.tobytes() == want.tobytes()
    assert portfolio_rollup(ylts[:1]) is ylts[0]
    with pytest.raises(ValueError):
        portfolio_rollup([])


def _same(a: float, b: float) -> bool:
    return (np.isnan(a) and np.isnan(b)) or a == b


@pytest.mark.parametrize("case", ["tiny", "many_rps", "signed_zeros", "nan_tail", "uniform", "all_equal"])
def test_k3_edge_cases(case, rng):
    """Shapes the radix select treats specially: one/two trials, more return
    periods than one launch holds (8) with duplicates sharing a prefix row,
    -0.0 next to +0.0, NaN (sorted last, like np.partition), no ties."""
    rps = [2.0, 10.0, 100.0, 250.0]
    if case == "tiny":
        x = np.array([3.0, 1.0])
        rps = [2.0]
    elif case == "many_rps":
        x = rng.lognormal(5.0, 2.0, 50_000)
        x[rng.random(x.size) < 0.2] = 1234.5
        rps = [1.5, 2.0, 2.0, 3.0, 5.0, 10.0, 10.0, 20.0, 50.0, 100.0, 200.0, 250.0, 500.0, 1000.0,
               2000.0, 5000.0, 10_000.0, 25_000.0, 50_000.0, 7.0]
    elif case == "signed_zeros":
        x = np.where(rng.random(10_000) < 0.5, -0.0, 0.0)
        x[:100] = rng.random(100)
    elif case == "nan_tail":
        x = rng.random(10_000)
        x[rng.choice(10_000, 30, replace=False)] = np.nan
        rps = [2.0, 100.0, 1000.0, 5000.0]
    elif case == "uniform":
        x = rng.random(300_000) * 1e5
    else:
        x = np.full(70_000, 42.0)
    p, t = order_stats(x, rps)
    for r, pv, tv in zip(rps, p, t):
        assert _same(pv, oracle.pml(x, r)), (r, pv, oracle.pml(x, r))
        want = oracle.tvar(x, r)
        assert (np.isnan(tv) and np.isnan(want)) or tv == pytest.approx(want, rel=1e-12, abs=1e-300)


def test_ep_curve_many_points_one_sort(rng):
    """Many return periods: one device sort of the keys (are_pml_many_device)
    -- the reference's own one-sort EP curve (metrics.py:97-115) -- exact
    points, including ties at a cap, negative zero and NaN (sorted last)."""
    import torch

    x = np.minimum(rng.lognormal(8.0, 2.0, 1_000_000), 66_000.0)
    x[rng.integers(0, x.size, 1000)] = 0.0
    x[:3] = [-0.0, np.nan, 1e300]
    rps = np.unique(np.concatenate([np.geomspace(1.01, 1e6, 97), [2.0, 10.0, 1e6]]))
    want = oracle.ep_points(x, rps)
    assert len(want) == rps.size and not any(np.isnan(a) for a, _ in want)  # NaN sorts past every rank asked
    got = ep_curve(YearLossTable("x", x), rps)
    assert list(got.points) == list(want)
    assert np.signbit(got.points[0][0]) == np.signbit(want[0][0])
    assert list(ep_curve(torch.from_numpy(x).cuda(), rps).points) == list(want)


def test_summary_mean_and_max_ride_in_k3(rng):
    import torch

    from paper_1308_2066_b200.risk import order_stats_summary

    x = rng.lognormal(6.0, 1.5, 300_001)
    p, t, mean, peak = order_stats_summary(torch.from_numpy(x).cuda(), [10.0, 100.0])
    assert list(p) == [oracle.pml(x, 10.0), oracle.pml(x, 100.0)]
    assert t[1] == pytest.approx(oracle.tvar(x, 100.0), rel=1e-12)
    assert peak == x.max() and mean == pytest.approx(x.mean(), rel=1e-13)
    y = x.copy()
    y[5] = np.nan
    _, _, mean, peak = order_stats_summary(torch.from_numpy(y).cuda(), [10.0])
    assert np.isnan(mean) and np.isnan(peak)


@pytest.mark.parametrize("max_ctas", [0, 2, 16])
def test_async_k3_on_a_few_ctas_matches(rng, max_ctas):
    """are_order_stats_async (pipelined callers: K3 on the SMs K2 leaves free,
    no host wait) against the blocking K3 and numpy: PML exact, TVaR rel
    1e-12 (its partial sums combine over a different grid)."""
    import torch

    from paper_1308_2066_b200.risk import order_stats_async

    x = np.minimum(rng.lognormal(8.0, 2.0, 300_001), 66_000.0)
    x[rng.integers(0, x.size, 500)] = 0.0
    d = torch.from_numpy(x).cuda()
    rps = [10.0, 50.0, 100.0, 250.0, 2.0]
    res = torch.zeros(16, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    order_stats_async(d, rps, res, side, max_ctas=max_ctas)
    side.synchronize()
    got = res.cpu().numpy()
    p, t = order_stats(d, rps)
    for r, rp in enumerate(rps):
        assert got[r] == p[r] == oracle.pml(x, rp)
        ref = oracle.tvar(x, rp)
        assert abs(got[8 + r] - ref) <= 1e-12 * abs(ref)
    with pytest.raises(ValueError):
        order_stats_async(d, [10.0] * 9, res, side)
    with pytest.raises(ValueError):
        order_stats_async(d, [0.5], res, side)


def test_ep_curve_runs_of_near_equal_losses(rng):
    """The EP sort orders by the keys' high 32 bits and resolves runs of equal
    high halves per requested rank: all-equal runs (a cap), short runs of
    distinct near-equal losses (counted), and long ones (the 64-bit sort
    fallback) must all give the exact order statistics."""
    n = 200_000

    def rp_at(arr, value, offset):
        # a return period whose rank k = n - floor(n / rp) lands `offset` into
        # the run starting at `value`
        k = int(np.searchsorted(np.sort(arr), value)) + 1 + offset
        return n / (n - k + 0.5)

    x = rng.lognormal(6.0, 1.0, n)
    x[:50_000] = 7_000.0                                   # a tie run
    x[50_000:50_200] = 3_000.0 + np.arange(200) * 1e-9     # a short run, distinct low bits
    rps = np.unique(np.concatenate([np.geomspace(1.05, 2e5, 60),
                                    [rp_at(x, 3_000.0, o) for o in (0, 37, 199)], [rp_at(x, 7_000.0, 10)]]))
    got = ep_curve(YearLossTable("x", x), rps).points
    assert list(got) == list(oracle.ep_points(x, rps))
    assert any(3_000.0 < v < 3_000.001 and v != 3_000.0 for v, _ in got)  # the short run was hit
    y = x.copy()
    y[50_000:55_000] = 3_000.0 + np.arange(5_000) * 1e-10  # a long run: the fallback
    rps_y = np.unique(np.concatenate([rps, [rp_at(y, 3_000.0, o) for o in (1, 2_500, 4_999)]]))
    assert list(ep_curve(YearLossTable("y", y), rps_y).points) == list(oracle.ep_points(y, rps_y))
