"""bench.py's roofline arithmetic (CPU): per-launch algorithmic bytes come from
the records each kernel's launches passed over, the stricter one-pass figure
credits n once."""

import importlib.util
import os

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(REPO, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_roofline_per_launch_and_one_pass(bench):
    n, rec, steps = 10**8, 12, 4
    # phases: moments, histogram, scan, scatter, classify, finish, recursion_stats, misc
    ms = [0.07, 1.7, 0.1, 7.08, 4.5, 4.64, 0.0, 0.0]
    launches = [4, 8, 8, 8, 8, 12, 0, 0]
    records = [0, 2 * n * steps, 0, 2 * n * steps, 0, n * steps, 0, 0]
    roof, phase_ms = bench.roofline_from_phases(n, rec, ms, launches, steps, 4, records)
    assert roof["kernel"] == "k_scatter" and roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert roof["launches_per_step"] == 2 and roof["records_per_step"] == 2 * n
    assert roof["alg_bytes_per_launch"] == 2 * rec * n
    assert roof["launch_ms"] == pytest.approx(7.08 / steps / 2)
    assert roof["achieved"] == pytest.approx(2 * 2 * rec * n / (7.08 / steps / 1e3) / 1e9)
    assert roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"])
    assert roof["one_pass_frac"] == pytest.approx(roof["frac"] / 2)
    assert phase_ms["scatter"] == pytest.approx(7.08 / steps)


def test_roofline_without_record_counts_credits_one_pass(bench):
    n, rec, steps = 10**7, 12, 2
    ms = [0.04, 0.06, 0.02, 0.26, 0.25, 0.27, 0.0, 0.0]
    launches = [2, 2, 2, 2, 2, 2, 0, 0]
    roof, _ = bench.roofline_from_phases(n, rec, ms, launches, steps, 2, None)
    assert roof["kernel"] == "k_finish"
    assert roof["alg_bytes_per_launch"] == 2 * rec * n
    assert roof["one_pass_frac"] == pytest.approx(roof["frac"])
