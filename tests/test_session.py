"""Session layer (§8f next rows): snapshot format, CSV formatting, the
reference's double moments, and run_session on the GPU — byte-identical to
the reference's run_session artefacts (goldens from the unmodified reference)."""
import hashlib
import struct

import numpy as np
import pytest

import paper_1606_00310_b200 as octgpu
from paper_1606_00310_b200.session import (RunConfig, measurements_csv, parse_measurements_csv, reference_moments,
                                           run_session)
from paper_1606_00310_b200.snapshot import parse_snapshot, serialize_snapshot


def _oracle_state(oracle, X, Y, p, q, seed, mcs):
    from oracle import OracleLattice
    L = OracleLattice.flat(oracle, X, Y, seed)
    L.step(oracle, oracle.resolve(p), oracle.resolve(q), mcs)
    return L


def test_snapshot_bytes_match_reference(oracle, goldens):
    s = goldens["sessions"][0]  # 1024^2 p=0.5 seed 1 t=1000
    L = _oracle_state(oracle, s["X"], s["Y"], s["p"], s["q"], s["seed"], s["tmax"])
    f = octgpu.SlopeField(octgpu.LatticeConfig(s["X"], s["Y"]), L.planes, L.t, L.phase)
    data = serialize_snapshot(f, octgpu.RngStreamSet(s["seed"], L.states))
    assert len(data) == s["snap_bytes"]
    assert hashlib.sha256(data).hexdigest() == s["snap_sha256"]
    f2, st2 = parse_snapshot(data)
    assert f2 == f and np.array_equal(st2.states, L.states) and st2.master_seed == s["seed"]


def test_snapshot_w32_and_no_trailer_roundtrip():
    cfg = octgpu.LatticeConfig(128, 6, 32)
    f = octgpu.new_flat(cfg)
    f.planes[0, 2, 1] = 0x12345678
    f.t_mcs, f.phase = 77, 1
    f2, st = parse_snapshot(serialize_snapshot(f))
    assert st is None and f2 == f and f2.planes.dtype == np.uint32


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXXXXXX" + b[8:], "not a snapshot file (bad magic)"),
    (lambda b: b[:40], "snapshot truncated"),
    (lambda b: b[:28] + bytes([2]) + b[29:], "snapshot phase must be 0 or 1"),
    (lambda b: b[:29] + bytes([0]) + b[30:], "unsupported bit convention flag 0"),
    (lambda b: b + b"junkjunk", "unrecognized trailing bytes after planes"),
    (lambda b: b[:8] + struct.pack("<I", 100) + b[12:], "snapshot header invalid: X must be a positive multiple"),
])
def test_snapshot_errors(mutate, msg):
    f = octgpu.new_flat(octgpu.LatticeConfig(128, 4))
    with pytest.raises(octgpu.IoError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        parse_snapshot(mutate(serialize_snapshot(f)))


def test_csv_format_roundtrip(goldens):
    for s in goldens["sessions"]:
        recs = parse_measurements_csv(s["csv"])
        cfg = RunConfig(X=s["X"], Y=s["Y"], w=s["w"], p=s["p"], q=s["q"], seed=s["seed"], t_max=s["tmax"],
                        ppd=s["ppd"])
        assert measurements_csv(cfg, recs) == s["csv"]


def test_reference_double_moments_bit_exact(oracle):
    L = _oracle_state(oracle, 512, 64, 0.5, 0.25, 3, 40)
    h, _ = oracle.reconstruct(L.planes)
    rec = reference_moments(40, h)
    m = oracle.height_moments(h)
    assert (rec.mean_h, rec.W2, rec.skew, rec.kurt) == (m[0], m[1], m[4], m[5])


def test_growth_fit_runs():
    from paper_1606_00310_b200.session import growth_exponent_fit
    recs = [octgpu.MeasurementRecord(t, 0.3 * t ** 0.48, 0, 0, 0) for t in (1, 2, 4, 8, 16, 32, 64)]
    fit = growth_exponent_fit(recs, 1, 64)
    assert abs(fit["beta"] - 0.24) < 1e-12 and fit["points"] == 7


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [0, 1, 2])
def test_run_session_byte_identical(goldens, tmp_path, idx):
    s = goldens["sessions"][idx]
    cfg = RunConfig(X=s["X"], Y=s["Y"], w=s["w"], p=s["p"], q=s["q"], seed=s["seed"], t_max=s["tmax"],
                    ppd=s["ppd"], out_dir=str(tmp_path))
    res = run_session(cfg)
    assert open(res.csv_path).read() == s["csv"]
    assert hashlib.sha256(open(res.snapshot_path, "rb").read()).hexdigest() == s["snap_sha256"]


@pytest.mark.gpu
def test_run_session_resume_and_exact_moments(goldens, tmp_path):
    s = goldens["sessions"][0]
    a = RunConfig(X=s["X"], Y=s["Y"], p=s["p"], q=s["q"], seed=s["seed"], t_max=100, ppd=s["ppd"],
                  out_dir=str(tmp_path / "a"))
    run_session(a)
    b = RunConfig(X=s["X"], Y=s["Y"], p=s["p"], q=s["q"], seed=s["seed"], t_max=s["tmax"], ppd=s["ppd"],
                  out_dir=str(tmp_path / "b"), resume=str(tmp_path / "a" / "final.snap"), moments="exact")
    res = run_session(b)
    assert hashlib.sha256(open(res.snapshot_path, "rb").read()).hexdigest() == s["snap_sha256"]
    ref = {r.t: r for r in parse_measurements_csv(s["csv"])}
    for r in res.records:
        assert r.mean_h == ref[r.t].mean_h
        assert abs(r.W2 - ref[r.t].W2) <= s["X"] * s["Y"] * 2.0 ** -52 * ref[r.t].W2


def test_cli_config_errors_exit_1():
    from paper_1606_00310_b200.__main__ import main
    assert main(["run", "--size", "1000", "--p", "0.5"]) == 1
    assert main(["run", "--size", "1024", "--p", "1.5"]) == 1
    assert main(["run", "--x", "256", "--y", "3"]) == 1


@pytest.mark.gpu
def test_cli_run_matches_reference_session(goldens, tmp_path, capsys):
    from paper_1606_00310_b200.__main__ import main
    s = goldens["sessions"][1]  # p=1 q=0 1024^2 seed 1
    rc = main(["run", "--size", str(s["X"]), "--p", str(s["p"]), "--q", str(s["q"]), "--seed", str(s["seed"]),
               "--tmax", str(s["tmax"]), "--ppd", str(s["ppd"]), "--out", str(tmp_path)])
    assert rc == 0
    assert open(tmp_path / "measurements.csv").read() == s["csv"]
    assert main(["bench", "--size", "4096", "--p", "0.5", "--mcs", "200"]) == 0


@pytest.mark.gpu
def test_counter_rng_session_resume(tmp_path):
    """Opt-in counter rng through the session driver and CLI: a resumed run continues bit-exactly
    (the counter streams depend only on (seed, t, row)) and the metadata names the generator."""
    import json

    from paper_1606_00310_b200.__main__ import main
    kw = dict(X=512, Y=256, p=0.5, q=0.0, seed=3, ppd=4, rng="counter")
    whole = run_session(RunConfig(t_max=200, out_dir=str(tmp_path / "whole"), **kw))
    run_session(RunConfig(t_max=60, out_dir=str(tmp_path / "a"), **kw))
    resumed = run_session(RunConfig(t_max=200, out_dir=str(tmp_path / "b"), resume=str(tmp_path / "a" / "final.snap"),
                                    **kw))
    assert open(whole.snapshot_path, "rb").read() == open(resumed.snapshot_path, "rb").read()
    meta = json.load(open(whole.metadata_path))
    assert meta["rng"]["generator"] == "splitmix64-counter"
    xo = run_session(RunConfig(t_max=200, out_dir=str(tmp_path / "xo"), **{**kw, "rng": "xoshiro"}))
    assert open(xo.snapshot_path, "rb").read() != open(whole.snapshot_path, "rb").read()
    assert main(["bench", "--size", "4096", "--p", "0.5", "--mcs", "200", "--rng", "counter"]) == 0


@pytest.mark.gpu
def test_cli_bench_report_fields(capsys):
    """BenchReport: the x1 byte identity, gpus, the median of the repeats, the engine's own
    kernel plan, and the refusal of runs too short to time (< 1 ms)."""
    import json

    from paper_1606_00310_b200.__main__ import main
    capsys.readouterr()
    assert main(["bench", "--size", "4096", "--p", "0.5", "--mcs", "300", "--repeats", "3"]) == 0
    row = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert row["gpus"] == 1 and row["repeats"] == 3 and row["mcs"] == 300
    assert row["net_GBps"] == row["updates_per_ns"] * 1.0
    assert abs(row["updates_per_ns"] - 4096 * 4096 * 300 / (row["wall_s"] * 1e9)) < 1e-6 * row["updates_per_ns"]
    assert row["kernel"] in ("k_mcs_bulk", "k_mcs_deep") and row["mcs_per_launch"] >= 1
    assert main(["bench", "--size", "256", "--p", "0.5", "--mcs", "10", "--repeats", "1"]) == 1  # ~0.1 ms
