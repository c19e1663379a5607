"""run_session on the GPU engine, mirroring session.hpp / session.cpp:37-203.

Writes the same artefacts as the reference: measurements.csv (identical
header and %.17g records), final.snap (OCTSCA01 + OCTRNG01) and
metadata.json. With moments="reference" (default up to 2^26 sites) every
record is measure_heights on the device-reconstructed HeightMap with the
reference's sequential double accumulation, so the CSV is byte-identical to
the reference's; moments="exact" uses the device reduction (exact int128
sums; doubles within N*2^-52 of the reference's, no HeightMap download).
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from ._lib import ConfigError, IoError, lib
from .engine import GpuEngine, MeasurementRecord
from .params import LatticeConfig, ProbMode, UpdateParams, log_schedule
from .snapshot import load_snapshot, serialize_snapshot, write_file

VERSION = "0.1.0"  # octsca kVersion (version.hpp:5): the CSV header carries it


@dataclass
class RunConfig:
    """session.hpp:14-39 (engine "gpu" added; workers accepted and ignored)."""

    X: int = 0
    Y: int = 0
    w: int = 64
    p: float = 0.5
    q: float = 0.0
    pmode: ProbMode | None = None
    qmode: ProbMode | None = None
    seed: int = 1
    workers: int = 1
    t_max: int = 1000
    ppd: int = 8
    engine: str = "gpu"
    out_dir: str = "."
    resume: str = ""
    fit_window: tuple | None = None
    moments: str = "auto"  # "reference" | "exact" | "auto"
    device: int = 0
    rng: str = "xoshiro"  # "xoshiro" (the reference's streams) | "counter" (opt-in, GpuEngine.set_rng)

    def update_params(self) -> UpdateParams:
        return UpdateParams.make(self.p, self.q, self.pmode, self.qmode)

    def lattice(self) -> LatticeConfig:
        return LatticeConfig(self.X, self.Y, self.w)

    def validate(self) -> None:  # session.cpp:89-100
        self.lattice().validate()
        if self.engine != "gpu":
            raise ConfigError(f"engine must be 'gpu', got '{self.engine}'")
        if self.workers < 1:
            raise ConfigError("workers must be >= 1")
        if self.t_max < 1:
            raise ConfigError("tmax must be >= 1")
        self.update_params()
        if self.fit_window and self.fit_window[0] >= self.fit_window[1]:
            raise ConfigError("fit window must satisfy tmin < tmax")
        if self.moments not in ("auto", "reference", "exact"):
            raise ConfigError(f"moments must be auto, reference or exact, got '{self.moments}'")


@dataclass
class SessionResult:
    records: list
    csv_path: str
    snapshot_path: str
    metadata_path: str
    fit: dict | None = None
    wall_s: float = 0.0
    extra: dict = field(default_factory=dict)


def reference_moments(t: int, heights: np.ndarray) -> MeasurementRecord:
    """measure_heights (measure.cpp:53-56) with the reference's double arithmetic."""
    Y, X = heights.shape
    out = (C.c_double * 6)()
    h = np.ascontiguousarray(heights, np.int32)
    lib().octgpu_height_moments(X, Y, h.ctypes.data_as(C.c_void_p), out)
    return MeasurementRecord(t, out[1], out[0], out[4], out[5], X * Y)


def _fmt_g17(v: float) -> str:
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def measurements_csv(cfg: RunConfig, records) -> str:
    """session.cpp:102-117."""
    prm = cfg.update_params()
    lines = [f"# octsca measurements v{VERSION}",
             f"# seed={cfg.seed} X={cfg.X} Y={cfg.Y} w={cfg.w} p={'%g' % cfg.p} pmode={prm.p.mode.label} "
             f"q={'%g' % cfg.q} qmode={prm.q.mode.label} tmax={cfg.t_max} ppd={cfg.ppd}",
             "t,W2,mean_h,skew,kurt"]
    for r in records:
        lines.append(f"{r.t},{_fmt_g17(r.W2)},{_fmt_g17(r.mean_h)},{_fmt_g17(r.skew)},{_fmt_g17(r.kurt)}")
    return "\n".join(lines) + "\n"


def parse_measurements_csv(text: str) -> list[MeasurementRecord]:
    """session.cpp:119-140."""
    out = []
    for line in text.splitlines():
        if not line or line[0] == "#" or line.startswith("t,"):
            continue
        parts = line.split(",")
        if len(parts) != 5:
            raise IoError(f"malformed measurement line: {line}")
        out.append(MeasurementRecord(int(parts[0]), *(float(x) for x in parts[1:])))
    return out


def linear_fit(xs, ys) -> dict:
    """measure.cpp:58-89."""
    n = len(xs)
    if n != len(ys) or n < 2:
        raise ConfigError("linear fit needs at least 2 points")
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    syy = sum((y - my) ** 2 for y in ys)
    if sxx == 0.0:
        raise ConfigError("linear fit is degenerate: all x equal")
    slope = sxy / sxx
    icpt = my - slope * mx
    ssr = sum((y - (slope * x + icpt)) ** 2 for x, y in zip(xs, ys))
    return {"slope": slope, "intercept": icpt, "r2": 1.0 if syy == 0.0 else 1.0 - ssr / syy,
            "stderr_slope": math.sqrt(ssr / (n - 2) / sxx) if n > 2 else 0.0, "n": n}


def growth_exponent_fit(records, t_min: int, t_max: int) -> dict:
    """measure.cpp:105-127: beta = slope of log W against log t."""
    sel = [r for r in records if t_min <= r.t <= t_max and r.t > 0 and r.W2 > 0]
    if len(sel) < 5:
        raise ConfigError(f"growth fit needs >= 5 records in window, have {len(sel)}")
    lf = linear_fit([math.log(r.t) for r in sel], [0.5 * math.log(r.W2) for r in sel])
    return {"beta": lf["slope"], "stderr": lf["stderr_slope"], "r2": lf["r2"], "t_min": t_min, "t_max": t_max,
            "points": lf["n"]}


def run_session(cfg: RunConfig) -> SessionResult:
    """session.cpp:142-203 on the GPU engine."""
    cfg.validate()
    prm = cfg.update_params()
    schedule = log_schedule(cfg.t_max, cfg.ppd)
    try:
        os.makedirs(cfg.out_dir, exist_ok=True)
    except OSError as e:
        raise IoError(f"cannot create output directory {cfg.out_dir}: {e}") from None
    moments = cfg.moments
    if moments == "auto":
        moments = "reference" if cfg.X * cfg.Y <= (1 << 26) else "exact"
    t0 = time.perf_counter()
    if cfg.resume:
        f, streams = load_snapshot(cfg.resume)
        if streams is None:
            raise ConfigError("snapshot has no RNG trailer; cannot resume bit-exactly")
        if f.cfg.w != cfg.w:
            raise ConfigError("snapshot word size does not match requested w")
        eng = GpuEngine(f, streams, device=cfg.device)
    else:
        eng = GpuEngine(cfg.lattice(), cfg.seed, device=cfg.device)
    eng.set_rng(cfg.rng)
    records = []
    for target in schedule:  # run.hpp:18-38
        if target < eng.t:
            continue
        if eng.t < target:
            eng.step(prm, target - eng.t)
        records.append(reference_moments(eng.t, eng.heights().h) if moments == "reference" else eng.measure())
    snap = serialize_snapshot(eng.field(), eng.streams())
    wall = time.perf_counter() - t0
    res = SessionResult(records, os.path.join(cfg.out_dir, "measurements.csv"),
                        os.path.join(cfg.out_dir, "final.snap"), os.path.join(cfg.out_dir, "metadata.json"),
                        wall_s=wall)
    write_file(res.csv_path, measurements_csv(cfg, records))
    write_file(res.snapshot_path, snap)
    if cfg.fit_window:
        res.fit = growth_exponent_fit(records, *cfg.fit_window)
    meta = {
        "tool": "octsca", "version": VERSION, "seed": cfg.seed, "engine": cfg.engine, "workers": cfg.workers,
        "lattice": {"X": cfg.X, "Y": cfg.Y, "w": cfg.w},
        "params": {"p": cfg.p, "pmode": prm.p.mode.label, "p_words": prm.p.draws_per_word(cfg.w),
                   "q": cfg.q, "qmode": prm.q.mode.label, "q_words": prm.q.draws_per_word(cfg.w)},
        "schedule": {"t_max": cfg.t_max, "points_per_decade": cfg.ppd, "times": schedule},
        "rng": ({"generator": "xoshiro256++", "streams": cfg.Y, "assignment": "one stream per lattice row"}
                if cfg.rng == "xoshiro" else
                {"generator": "splitmix64-counter", "streams": cfg.Y,
                 "assignment": "one counter stream per (sweep, row), keyed by the seed (opt-in, not the reference's)"}),
        "resume": cfg.resume,
        "outputs": {"measurements": res.csv_path, "snapshot": res.snapshot_path},
        "moments": moments,
        "device": lib().octgpu_version().decode(),
    }
    if res.fit:
        meta["fit"] = res.fit
    meta["wall_s"] = wall
    write_file(res.metadata_path, json.dumps(meta, indent=2) + "\n")
    return res
