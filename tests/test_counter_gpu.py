"""GPU counter-based rng mode (octgpu_set_rng, k_sweep_ctr) against the oracle's
oo_step_ctr: planes bit-exact, t / phase equal, xoshiro states untouched, and
mode switches mid-run (ghost rows and lazily owed xoshiro draws stay right)."""
import numpy as np
import pytest

import paper_1606_00310_b200 as octgpu
from oracle import OracleLattice

pytestmark = pytest.mark.gpu

GEOMS = [(128, 2, 64), (256, 34, 64), (1024, 94, 64), (1152, 262, 64), (2048, 482, 64), (64, 34, 32),
         (192, 66, 32)]
MODES = [(0.5, 0.0), (0.75, 0.0), (0.5, 0.5), (0.98, 0.02), (1.0, 0.0), (0.8125, 0.25), (0.0, 0.0)]


def _pair(oracle, X, Y, w, seed):
    eng = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y, w), seed)
    eng.set_rng("counter")
    return eng, OracleLattice.flat(oracle, X, Y, seed, w)


@pytest.mark.parametrize("deep", ["1", "2"], ids=["policy", "deep"])
@pytest.mark.parametrize("geom", GEOMS, ids=lambda g: f"{g[0]}x{g[1]}w{g[2]}")
@pytest.mark.parametrize("pq", MODES, ids=lambda m: f"p{m[0]}q{m[1]}")
def test_counter_vs_oracle(oracle, monkeypatch, deep, geom, pq):
    """deep=2 forces the 2-MCS pass (k_mcs_deep<CTR>) wherever the lattice takes it (n >= 8, >= 256 rows)."""
    monkeypatch.setenv("OCTGPU_DEEP", deep)
    X, Y, w = geom
    p, q = pq
    seed = 77 + X + Y
    eng, L = _pair(oracle, X, Y, w, seed)
    st0 = eng.streams().states.copy()
    prm = octgpu.UpdateParams.make(p, q)
    op, oq = oracle.resolve(p), oracle.resolve(q)
    for chunk in (1, 3, 4):
        eng.step(prm, chunk)
        L.step_ctr(oracle, op, oq, seed, chunk)
        assert np.array_equal(eng.planes(), L.planes.astype(eng.planes().dtype)), (chunk, eng.t)
        assert eng.t == L.t and eng.phase == L.phase
    assert np.array_equal(eng.streams().states, st0)
    assert eng.rng == "counter"


@pytest.mark.parametrize("deep", ["1", "2"], ids=["policy", "deep"])
@pytest.mark.parametrize("pq", [(0.5, 0.0), (1.0, 0.0), (0.98, 0.02)])
def test_mode_switch_mid_run(oracle, monkeypatch, deep, pq):
    """xoshiro -> counter -> xoshiro on a lattice the TMA kernels run (ghost rows refreshed after the
    in-place counter sweeps; constant-xi draws owed to the streams survive the switch)."""
    monkeypatch.setenv("OCTGPU_DEEP", deep)
    X, Y, seed = 1024, 262, 5
    p, q = pq
    eng = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), seed)
    L = OracleLattice.flat(oracle, X, Y, seed)
    prm = octgpu.UpdateParams.make(p, q)
    op, oq = oracle.resolve(p), oracle.resolve(q)
    eng.step(prm, 4)
    L.step(oracle, op, oq, 4)
    eng.set_rng("counter")
    eng.step(prm, 3)
    L.step_ctr(oracle, op, oq, seed, 3)
    eng.set_rng("xoshiro")
    eng.step(prm, 5)
    L.step(oracle, op, oq, 5)
    assert np.array_equal(eng.planes(), L.planes)
    assert np.array_equal(eng.streams().states, L.states)
    assert eng.t == L.t == 12


def test_counter_mode_errors():
    eng = octgpu.GpuEngine(octgpu.LatticeConfig(256, 34), 3)
    eng.set_rng("counter")
    with pytest.raises(octgpu.ConfigError):
        eng.sweep(0, octgpu.UpdateParams.make(0.5, 0.0))
    with pytest.raises(ValueError):
        eng.set_rng("philox")
    from paper_1606_00310_b200.stripes import StripeEngine
    st = StripeEngine(octgpu.LatticeConfig(256, 64), 0, 32, 3)
    with pytest.raises(octgpu.ConfigError):
        from paper_1606_00310_b200._lib import lib
        from paper_1606_00310_b200.engine import check
        check(lib().octgpu_set_rng(st._h, 1))


def test_counter_measure_consistent():
    """measure() after counter steps: the device's exact power sums equal the host reconstruction's."""
    eng = octgpu.GpuEngine(octgpu.LatticeConfig(512, 256), 9)
    eng.set_rng("counter")
    eng.step(octgpu.UpdateParams.make(0.5, 0.0), 40)
    rec = eng.measure()
    h = eng.heights().h.astype(np.int64)
    assert [int(v) for v in rec.power_sums[:2]] == [int(h.sum()), int((h * h).sum())]
    assert rec.W2 > 0.5


@pytest.mark.parametrize("deep", ["0", "2"], ids=["bulk", "deep"])
@pytest.mark.parametrize("pq", [(0.5, 0.0), (0.5, 0.5), (0.98, 0.02), (0.75, 0.25)])
def test_fused_counter_kernel_matches_sweeps(monkeypatch, deep, pq):
    """At sizes the oracle cannot reach: the fused TMA passes (k_mcs_bulk<CTR>, and k_mcs_deep<CTR> with
    deep=2 where the modes allow) equal two in-place k_sweep_ctr sweeps per MCS (OCTGPU_MCS_IMPL=1)."""
    X = Y = 4096
    prm = octgpu.UpdateParams.make(*pq)
    mcs = 3 if pq[0] == 0.98 else 21
    monkeypatch.setenv("OCTGPU_DEEP", deep)
    fused = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), 11)
    fused.set_rng("counter")
    fused.step(prm, mcs)
    monkeypatch.setenv("OCTGPU_MCS_IMPL", "1")
    plain = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), 11)
    plain.set_rng("counter")
    plain.step(prm, mcs)
    assert fused.checksum() == plain.checksum()
    assert np.array_equal(fused.planes(), plain.planes())


@pytest.mark.parametrize("deep", ["1", "2"], ids=["policy", "deep"])
@pytest.mark.parametrize("pq", [(0.5, 0.0), (0.5, 0.5), (1.0, 0.0)])
def test_counter_tile_shift_neutral(monkeypatch, deep, pq):
    """DTr-style tile-origin shifts move block / warp / halo boundaries; the counter streams are keyed by the
    lattice row, so the trajectory is unchanged."""
    monkeypatch.setenv("OCTGPU_DEEP", deep)
    cfg = octgpu.LatticeConfig(2048, 482)
    prm = octgpu.UpdateParams.make(*pq)
    a = octgpu.GpuEngine(cfg, 4)
    b = octgpu.GpuEngine(cfg, 4)
    for e in (a, b):
        e.set_rng("counter")
    b.set_tile_shift(12345)
    a.step(prm, 9)
    b.step(prm, 9)
    assert np.array_equal(a.planes(), b.planes())
