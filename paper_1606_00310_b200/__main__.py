"""Command line, following the reference's specified CLI:

    python -m paper_1606_00310_b200 run   --size 1024 --p 0.5 --q 0 --tmax 1000 --seed 42 --out DIR
    python -m paper_1606_00310_b200 bench --size 16384 --p 0.5 --mcs 100 [--csv]
    python -m paper_1606_00310_b200 fit   DIR/measurements.csv --tmin 50 --tmax 2000

Flags: --size/-L, --x, --y, --w, --p, --q, --pmode, --qmode, --seed, --workers,
--tmax, --ppd, --engine gpu, --out, --resume, --moments. Environment
overrides use the OCTSCA_ prefix (e.g. OCTSCA_SEED). Exit codes: 0 ok,
1 config error, 2 invariant violation, 3 I/O, 4 CUDA.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

from ._lib import OctError
from .params import ProbMode


def _env(name, default):
    return os.environ.get("OCTSCA_" + name.upper(), default)


def _mode(s):
    return None if s in (None, "", "auto") else ProbMode[s.capitalize()]


def _common(ap):
    ap.add_argument("--size", "-L", type=int, default=int(_env("size", 0)))
    ap.add_argument("--x", type=int, default=int(_env("x", 0)))
    ap.add_argument("--y", type=int, default=int(_env("y", 0)))
    ap.add_argument("--w", type=int, default=int(_env("w", 64)))
    ap.add_argument("--p", type=float, default=float(_env("p", 0.5)))
    ap.add_argument("--q", type=float, default=float(_env("q", 0.0)))
    ap.add_argument("--pmode", default=_env("pmode", "auto"))
    ap.add_argument("--qmode", default=_env("qmode", "auto"))
    ap.add_argument("--seed", type=int, default=int(_env("seed", 1)))
    ap.add_argument("--workers", type=int, default=int(_env("workers", 1)))
    ap.add_argument("--engine", default=_env("engine", "gpu"))
    ap.add_argument("--device", type=int, default=int(_env("device", 0)))
    ap.add_argument("--rng", default=_env("rng", "xoshiro"), choices=["xoshiro", "counter"],
                    help="xi source: the reference's xoshiro256++ streams, or opt-in counter-based streams")


def _dims(a):
    X = a.x or a.size
    Y = a.y or a.size
    return X, Y


def cmd_run(a) -> int:
    from .session import RunConfig, run_session

    X, Y = _dims(a)
    cfg = RunConfig(X=X, Y=Y, w=a.w, p=a.p, q=a.q, pmode=_mode(a.pmode), qmode=_mode(a.qmode), seed=a.seed,
                    workers=a.workers, t_max=a.tmax, ppd=a.ppd, engine=a.engine, out_dir=a.out, resume=a.resume,
                    moments=a.moments, device=a.device, rng=a.rng,
                    fit_window=(a.fit_tmin, a.fit_tmax) if a.fit_tmin is not None else None)
    res = run_session(cfg)
    print(json.dumps({"records": len(res.records), "csv": res.csv_path, "snapshot": res.snapshot_path,
                      "wall_s": res.wall_s, "fit": res.fit}))
    return 0


def cmd_bench(a) -> int:
    """BenchReport: engine,L,p,q,mode,workers,gpus,mcs,updates_per_ns,net_GBps,wall_s, the
    median over --repeats timed runs after a 10% warm-up; runs shorter than 1 ms in total are
    refused. The CPU reference column lives in bench.py (cpu_baseline / --impl reference): the
    reference engine is test infrastructure and the package never loads it."""
    from .engine import GpuEngine
    from .params import LatticeConfig, UpdateParams

    X, Y = _dims(a)
    prm = UpdateParams.make(a.p, a.q, _mode(a.pmode), _mode(a.qmode))
    eng = GpuEngine(LatticeConfig(X, Y, a.w), a.seed, device=a.device)
    eng.set_rng(a.rng)
    warm = max(1, a.mcs // 10)  # first 10% discarded
    eng.step(prm, warm)
    eng.sync()
    walls = []
    for _ in range(max(1, a.repeats)):
        t0 = time.perf_counter()
        eng.step(prm, a.mcs)
        eng.sync()
        walls.append(time.perf_counter() - t0)
    wall = sorted(walls)[len(walls) // 2]
    if wall < 1e-3:
        print(f"error: {a.mcs} MCS of {X}x{Y} took {wall * 1e3:.3f} ms < 1 ms: too short to time "
              f"(raise --mcs)", file=sys.stderr)
        return 1
    ups = X * Y * a.mcs / (wall * 1e9)
    kernel, mcs_per_launch = eng.pass_plan(prm)
    row = {"engine": "gpu" if a.rng == "xoshiro" else "gpu-counter-rng", "L": X if X == Y else f"{X}x{Y}",
           "p": a.p, "q": a.q,
           "mode": f"{prm.p.mode.label}/{prm.q.mode.label}", "workers": a.workers, "gpus": 1, "mcs": a.mcs,
           "updates_per_ns": ups, "net_GBps": ups * 1.0, "wall_s": wall, "repeats": len(walls),
           "kernel": kernel, "mcs_per_launch": mcs_per_launch}
    if a.csv:
        print(",".join(row))
        print(",".join(str(v) for v in row.values()))
    else:
        print(json.dumps(row))
    return 0


def cmd_fit(a) -> int:
    from .session import growth_exponent_fit, parse_measurements_csv
    from .snapshot import read_file

    recs = parse_measurements_csv(read_file(a.csv_path).decode())
    print(json.dumps(growth_exponent_fit(recs, a.tmin, a.tmax)))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="octsca-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    _common(r)
    r.add_argument("--tmax", type=int, default=int(_env("tmax", 1000)))
    r.add_argument("--ppd", type=int, default=int(_env("ppd", 8)))
    r.add_argument("--out", default=_env("out", "."))
    r.add_argument("--resume", default=_env("resume", ""))
    r.add_argument("--moments", default=_env("moments", "auto"))
    r.add_argument("--fit-tmin", type=int, default=None)
    r.add_argument("--fit-tmax", type=int, default=None)
    b = sub.add_parser("bench")
    _common(b)
    b.add_argument("--mcs", type=int, default=100)
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--csv", action="store_true")
    f = sub.add_parser("fit")
    f.add_argument("csv_path")
    f.add_argument("--tmin", type=int, required=True)
    f.add_argument("--tmax", type=int, required=True)
    a = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "bench": cmd_bench, "fit": cmd_fit}[a.cmd](a)
    except OctError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.exit_code


if __name__ == "__main__":
    sys.exit(main())
