"""Drop-in check: the reference's own driver code (octsca::run, measurements_csv,
serialize_snapshot, load_snapshot) running octsca::GpuEngine (the C++ header
over the C-ABI) must produce byte-identical session artefacts to the
reference's run_session with VecEngine (goldens from the unmodified reference)."""
import hashlib
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin")


def _run(args, tmp):
    if not os.path.exists(DROPIN):
        pytest.skip("oracle/_ref/dropin not built (needs the reference headers at build time)")
    r = subprocess.run([DROPIN] + [str(a) for a in args] + [str(tmp)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r


def _sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_session_artefacts_byte_identical(goldens, tmp_path, idx):
    s = goldens["sessions"][idx]
    _run([s["X"], s["Y"], s["w"], s["p"], s["q"], s["seed"], s["tmax"], s["ppd"]], tmp_path)
    csv = open(tmp_path / "measurements.csv").read()
    assert csv == s["csv"]
    assert _sha(tmp_path / "final.snap") == s["snap_sha256"]


def test_resume_from_snapshot_is_bit_exact(goldens, tmp_path):
    s = goldens["sessions"][0]  # 1024^2 p=0.5 seed 1, t_max 1000
    a = tmp_path / "a"
    a.mkdir()
    _run([s["X"], s["Y"], s["w"], s["p"], s["q"], s["seed"], 316, s["ppd"]], a)
    b = tmp_path / "b"
    b.mkdir()
    args = [s["X"], s["Y"], s["w"], s["p"], s["q"], s["seed"], s["tmax"], s["ppd"], b, a / "final.snap"]
    r = subprocess.run([DROPIN] + [str(v) for v in args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert _sha(b / "final.snap") == s["snap_sha256"]
    # the resumed CSV is the tail of the uninterrupted one (run.hpp:27-29 skips past times)
    full = [l for l in s["csv"].splitlines() if l and l[0].isdigit()]
    tail = [l for l in open(b / "measurements.csv").read().splitlines() if l and l[0].isdigit()]
    assert tail == [l for l in full if int(l.split(",")[0]) >= 316]


STRIPES = os.path.join(ROOT, "oracle", "_ref", "stripes_dropin")


@pytest.mark.parametrize("X,Y,parts", [(2048, 256, 4), (1024, 130, 3), (4096, 512, 8)])
def test_cpp_stripe_group_matches_engine(X, Y, parts):
    """octsca::GpuStripeGroup (C++, peer-memory halos, native combine) == octsca::GpuEngine
    under the reference's own octsca::run, for constant and live parameter legs."""
    if not os.path.exists(STRIPES):
        pytest.skip("oracle/_ref/stripes_dropin not built (needs the reference headers at build time)")
    env = dict(os.environ, OCTGPU_DEEP="2")  # 2-MCS stripe passes at test sizes
    r = subprocess.run([STRIPES, str(X), str(Y), str(parts), "11"], capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("stripes ok")
