"""Bit-exact parity at the BASELINE geometries, under the DEFAULT kernel policy.

The engine runs exactly as the bench does (no OCTGPU_* overrides): at 2^16 x 2^16 and 2^17 x 2^17 the
production dispatch is k_mcs_deep (3 MCS per pass for constant xi from 2^28 sites, 2 MCS per pass for one
draw per word from 2^30) or k_mcs_bulk (1 MCS per pass), on the full 266- / 532-block grids with their ghost-row wrap and the
branch-free steady state of the deep pipeline (504 / 1016 iterations per row). Each case is compared with
the compiled reference VecEngine<uint64_t> (oracle/_ref, the unmodified reference on all host cores) on
the same seed: field_checksum (slope_field.hpp:232-246), the RNG-state digest of every row stream
(rng.hpp:80-94), t and phase after N MCS (engine_vec.hpp:171-177), and the exact height power sums
against the oracle's at-scale reconstruction (oo_measure_planes_mt: slope_field.hpp:206-229).
"""
import os

import numpy as np
import pytest

import paper_1606_00310_b200 as octgpu

pytestmark = pytest.mark.gpu

CORES = os.cpu_count() or 1


@pytest.fixture(autouse=True)
def _default_policy(monkeypatch):
    for k in list(os.environ):
        if k.startswith("OCTGPU_"):
            monkeypatch.delenv(k)


def _digest(oracle, states):
    return oracle.states_digest(np.ascontiguousarray(states, np.uint64))


# (name, X, Y, p, q, MCS, expected kernel launches): BASELINE configs 2' (p = 1/2, the paper's case), 3, 4, 2
# and 5; every k_mcs_deep pass is followed by the ghost-row copy kernel
CASES = [
    ("c2h", 1 << 16, 1 << 16, 0.5, 0.0, 20, 20),   # k_mcs_deep x 10, live xoshiro (one draw per word)
    ("c3", 1 << 16, 1 << 16, 0.5, 0.5, 10, 10),    # k_mcs_deep x 5, live xoshiro (two half draws per word)
    ("c4", 1 << 16, 1 << 16, 0.98, 0.02, 2, 2),    # k_mcs_bulk, arbitrary (128 draws per word)
    ("c2", 1 << 16, 1 << 16, 1.0, 0.0, 20, 12),    # k_mcs_deep, constant xi: 2 x 4 MCS + 4 x 3 MCS (lazy draws)
    ("c5h", 1 << 17, 1 << 17, 0.5, 0.0, 4, 4),     # k_mcs_deep x 2 at 2^34 sites
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_baseline_geometry_matches_reference(oracle, reflib, case):
    from oracle import RefEngine

    name, X, Y, p, q, mcs, passes = case
    seed = 1
    eng = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y, 64), seed)
    prm = octgpu.UpdateParams.make(p, q)
    l0 = eng.launches
    eng.step(prm, mcs)
    eng.sync()
    assert eng.launches - l0 == passes, "not the production kernel dispatch"
    gpu_sum = eng.checksum()
    gpu_states = eng.streams().states  # materialises lazily-owed draws (constant xi)
    rec = eng.measure()

    ref = RefEngine(reflib, X, Y, seed, workers=CORES)
    ref.step(p, q, mcs)
    assert (eng.t, eng.phase) == (ref.t, ref.phase) == (mcs, 0)
    assert gpu_sum == ref.checksum()
    assert _digest(oracle, gpu_states) == _digest(oracle, ref.states())
    sums, err = oracle.measure_planes(ref.planes())
    assert err is None
    assert list(rec.power_sums) == sums
    assert rec.mean_h == sums[0] / (X * Y)


# (name, X, Y, [(p, q, MCS), ...]): mixed schedules through the default dispatch -- p = 1 on a ROUGH field runs
# the 3-MCS constant-xi pass on non-trivial dynamics (from the flat start p = 1 returns to flat every MCS), and a
# long p = 1/2 leg checks the 2-MCS live pass over 100 passes
LEGS = [
    ("c2rough", 1 << 16, 1 << 16, [(0.5, 0.0, 6), (1.0, 0.0, 21), (0.5, 0.5, 3), (0.0, 0.0, 3)]),
    ("c2h200", 1 << 16, 1 << 16, [(0.5, 0.0, 200)]),
]


@pytest.mark.parametrize("case", LEGS, ids=[c[0] for c in LEGS])
def test_mixed_schedules_match_reference(oracle, reflib, case):
    from oracle import RefEngine

    name, X, Y, legs = case
    eng = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y, 64), 3)
    ref = RefEngine(reflib, X, Y, 3, workers=CORES)
    for p, q, mcs in legs:
        eng.step(octgpu.UpdateParams.make(p, q), mcs)
        ref.step(p, q, mcs)
    eng.sync()
    assert eng.checksum() == ref.checksum()
    assert _digest(oracle, eng.streams().states) == _digest(oracle, ref.states())
    sums, err = oracle.measure_planes(ref.planes())
    assert err is None and list(eng.measure().power_sums) == sums


def test_eight_peer_stripes_match_periodic_engine_2p17(oracle):
    """BASELINE configs[4]: the 2^17 x 2^17 lattice as 8 row stripes (SweepPlan blocks, params.hpp:107-127)
    exchanging halos device-side over peer memory, against the periodic engine: p = 1 (2-MCS stripe passes)
    then p = 1/2 (one-MCS passes, live streams), planes, rng states and exact moments bit-identical."""
    import torch

    from paper_1606_00310_b200.stripes import PeerLocalTransport, StripeEngine, StripeGroup, stripe_bounds

    X = Y = 1 << 17
    cfg = octgpu.LatticeConfig(X, Y)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        engines = []
        for r in range(8):
            y0, y1 = stripe_bounds(Y, 8, r)
            e = StripeEngine(cfg, y0, y1, 1)
            e.set_stream(stream.cuda_stream)
            engines.append(e)
        grp = StripeGroup(PeerLocalTransport(engines), X, Y)
        ref = octgpu.GpuEngine(cfg, 1)
        for pq, n in (((1.0, 0.0), 4), ((0.5, 0.0), 3)):
            prm = octgpu.UpdateParams.make(*pq)
            grp.step(prm, n)
            ref.step(prm, n)
        grp.sync()
        ref.sync()
        planes = np.concatenate([e.planes() for e in engines], axis=1)
        assert np.array_equal(planes, ref.planes())
        del planes
        states = np.concatenate([e.states() for e in engines], axis=0)
        assert np.array_equal(states, ref.streams().states)
        rec, rref = grp.measure(), ref.measure()
        assert rec.power_sums == rref.power_sums
        grp.tr.engines = []
        del grp, engines
