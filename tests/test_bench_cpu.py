"""bench.py's host logic without a GPU: the timed window over the 10^4-MCS job and the kernel labels
the roofline is computed for (mirrors of engine.cu's dispatch policy)."""
import os
import sys

import pytest

import paper_1606_00310_b200 as octgpu
from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402

SCHED = octgpu.log_schedule(10_000, 8)


def test_window_default_is_the_whole_job():
    t0, sched, targets, desc = bench.timed_window(10_000, False, SCHED)
    assert t0 == 0 and sched == SCHED and len(sched) == 33 and targets[-1] == 10_000
    assert "from the flat start" in desc


@pytest.mark.parametrize("K", [1, 3, 50, 999, 1000])
def test_short_window_is_the_end_of_the_job(K):
    t0, sched, targets, desc = bench.timed_window(K, False, SCHED)
    assert t0 == 10_000 - K and targets[-1] == 10_000
    assert all(t0 < t <= 10_000 for t in targets) and sched[-1] == 10_000
    assert f"state at t={t0} prepared untimed" in desc


def test_from_flat_and_beyond_the_job():
    t0, sched, targets, _ = bench.timed_window(30, True, SCHED)
    assert t0 == 0 and targets[-1] == 30 and sched == [t for t in SCHED if t <= 30]
    t0, sched, targets, desc = bench.timed_window(12_000, False, SCHED)
    assert t0 == 0 and targets[-1] == 12_000 and len(sched) == 33 and "2000 MCS more" in desc
