"""The C-ABI boundary without a GPU: the library loads, exports exactly what
include/octgpu.h declares, and its host-side logic (parameter resolution,
validation, stream seeding, schedules) matches the reference goldens."""
import os
import re

import numpy as np
import pytest

import paper_1606_00310_b200 as octgpu
from paper_1606_00310_b200 import _lib
from conftest import HAS_GPU, ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "octgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(octgpu_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    decl = _declared()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(decl) == sorted(_lib.EXPORTS)
    assert b"sm_100a" in L.octgpu_version()


def test_header_is_plain_c(tmp_path):
    """include/octgpu.h is the FFI boundary (ctypes, cgo, JNI): it must compile as strict C99."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    src = tmp_path / "t.c"
    src.write_text('#include "octgpu.h"\nint main(void) { octgpu_engine* e = 0; (void)e; '
                   'return OCTGPU_RNG_COUNTER - 1; }\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only",
                        "-I" + os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_library_is_sm100a_cubin():
    so = _lib.LIB_PATH
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_resolve_matches_reference(goldens):
    for case in goldens["resolve"]:
        forced = None if case["forced"] < 0 else case["forced"]
        if case["rc"]:
            with pytest.raises(octgpu.ConfigError) as ei:
                octgpu.ProbSpec.resolve(case["r"], forced)
            assert str(ei.value) == case["err"]
            continue
        s = octgpu.ProbSpec.resolve(case["r"], forced)
        assert int(s.mode) == case["mode"]
        assert s.draws_per_word(64) == case["draws"]
        if s.mode == octgpu.ProbMode.Dyadic:
            assert (s.plan.k, s.plan.m) == (case["k"], case["m"])


def test_validate_lattice_messages():
    with pytest.raises(octgpu.ConfigError, match="X must be a positive multiple of 2\\*w = 128, got 1000"):
        octgpu.LatticeConfig(1000, 1000).validate()
    with pytest.raises(octgpu.ConfigError, match="Y must be even and >= 2, got 3"):
        octgpu.LatticeConfig(128, 3).validate()
    with pytest.raises(octgpu.ConfigError, match="word size must be 32 or 64, got 16"):
        octgpu.LatticeConfig(128, 2, 16).validate()
    octgpu.LatticeConfig(64, 2, 32).validate()
    # construction validates before touching the device
    with pytest.raises(octgpu.ConfigError):
        octgpu.GpuEngine(octgpu.LatticeConfig(100, 4), 1)


def test_stream_states_match_oracle(oracle, goldens):
    for seed, n in [(1, 3), (42, 17), (0, 5), (2 ** 64 - 1, 9), (12345, 64)]:
        got = octgpu.RngStreamSet.derive(seed, n).states
        assert np.array_equal(got, oracle.stream_set(seed, n)), seed
    k = goldens["kat"]["stream_set_1_3"]
    got = octgpu.RngStreamSet.derive(1, 3).states
    assert [[int(v) for v in r] for r in got] == [[int(v, 16) for v in r] for r in k]


def test_log_schedule_matches_reference(goldens):
    for key, val in goldens["log_schedule"].items():
        t, p = map(int, key.split(","))
        assert octgpu.log_schedule(t, p) == val
    with pytest.raises(octgpu.ConfigError):
        octgpu.log_schedule(0, 8)


def test_update_params_draws():
    assert octgpu.UpdateParams.make(0.5, 0.0).draws_per_word() == 1
    assert octgpu.UpdateParams.make(0.5, 0.5).draws_per_word() == 2
    assert octgpu.UpdateParams.make(0.98, 0.02).draws_per_word() == 128
    assert octgpu.UpdateParams.make(1.0, 0.0).draws_per_word() == 64
    assert octgpu.UpdateParams.make(0.75, 0.0).draws_per_word(32) == 2
    assert octgpu.UpdateParams.make(0.95, 0.0).draws_per_word(32) == 32


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(octgpu.CudaError):
        octgpu.GpuEngine(octgpu.LatticeConfig(128, 2), 1)
