"""Every hot-set kernel over the parity suite.

The library runs k2_pair (two trials per warp) for launches whose mean trial
is short and the relay kernel otherwise (csrc/k2_trials.cu `use_pair`), so in
a normal run each parity test exercises one of them.  ARE_K2_PAIR=0/1 forces
one of the two for the whole process, and ARE_K2_RELAY=0 replaces the relay
kernel by the legacy k2_hotset (and k2_pair then reads the hot-set slots
instead of the relay records); this runs the core parity tests under each in
a subprocess so every kernel meets every case.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ("random_instances or plugin_run_trials or worked or empty_trial or c1_ylt or seed31 or nan_inf "
         "or large_catalogs or 256_tables or long_and_ragged or instantiations or resident_and_pinned")


@pytest.mark.parametrize("force,relay", [("0", "1"), ("0", "0"), ("1", "1"), ("1", "0")],
                         ids=["k2_relay", "k2_hotset", "k2_pair_relay_records", "k2_pair_slots"])
def test_parity_suite_under_each_kernel(force, relay):
    env = dict(os.environ, ARE_K2_PAIR=force, ARE_K2_RELAY=relay)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q",
                        "-x", "-p", "no:cacheprovider", "-k", CASES], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_dense_suite_under_lane_per_line_kernel():
    """ARE_DENSE_COOP=0 runs the lane-per-line event-major dense kernel
    (k2_dense<EM>) in place of the cooperative one: the dense parity tests
    under it, so the A/B path stays bit-exact too."""
    env = dict(os.environ, ARE_DENSE_COOP="0")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q",
                        "-x", "-p", "no:cacheprovider", "-k", "dense or degenerate or instantiations or 256_tables"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
