"""Driver loop mirroring ``octsca::run`` (run.hpp:18-38).

Advances the engine to every scheduled time and measures there. Scheduled
times already in the past are skipped (resumed runs, run.hpp:27-29). With a
GpuEngine the measurement is the device-side ``measure()``; any other engine
with a ``heights()`` method is measured through the host moments.
"""
from __future__ import annotations

from typing import Callable, Iterable

from ._lib import ConfigError
from .engine import MeasurementRecord


def run(eng, prm, schedule: Iterable[int], sink: Callable[[MeasurementRecord], None] | None = None,
        batch: bool = True) -> list[MeasurementRecord]:
    schedule = list(schedule)
    for i in range(1, len(schedule)):
        if schedule[i] <= schedule[i - 1]:
            raise ConfigError("schedule must be strictly increasing")
    records: list[MeasurementRecord] = []
    for target in schedule:
        if target < eng.t:
            continue
        if eng.t < target:
            if batch:
                eng.step(prm, target - eng.t)  # one enqueue of the whole stretch
            else:
                while eng.t < target:
                    eng.step(prm)
        rec = eng.measure()
        records.append(rec)
        if sink:
            sink(rec)
    return records
