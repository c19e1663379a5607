"""Opt-in counter-based rng mode (include/octgpu.h octgpu_set_rng; no reference
equivalent). CPU side: the oracle's generator against a
pure-Python restatement of its definition, draw statistics, and the oracle's
counter-mode sweeps (heights stay consistent, the surface roughens)."""
import numpy as np

from oracle import OracleLattice

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def ctr_draw(seed, sigma, y, i):
    key = mix64((seed + (sigma + 1) * GAMMA) & M64)
    origin = mix64((key + (y + 1) * GAMMA) & M64)
    return mix64((origin + (i + 1) * GAMMA) & M64)


def test_mix64_is_splitmix64_finaliser():
    # SplitMix64 from state 0: first output (Steele, Lea, Flood 2014; also the reference's seeding, rng.hpp)
    assert mix64(GAMMA) == 0xE220A8397B1DCDAF


def test_oracle_draws_match_definition(oracle):
    for seed, sigma, y, i in [(1, 0, 0, 0), (1, 0, 0, 1), (42, 7, 1023, 63), (M64, 2 * 10**4 + 1, 65535, 127),
                              (12345, 3, 17, 5000)]:
        assert oracle.ctr_draw(seed, sigma, y, i) == ctr_draw(seed, sigma, y, i)


def test_draw_bits_are_balanced(oracle):
    n = 4096
    words = np.array([oracle.ctr_draw(7, s, y, i) for s in range(2) for y in range(32) for i in range(n // 64)],
                     np.uint64)
    bits = np.unpackbits(words.view(np.uint8))
    frac = bits.mean()
    sd = 0.5 / np.sqrt(bits.size)
    assert abs(frac - 0.5) < 5 * sd
    # neighbouring rows and sweeps are not correlated bitwise
    a = np.array([oracle.ctr_draw(7, 0, 0, i) for i in range(512)], np.uint64)
    b = np.array([oracle.ctr_draw(7, 0, 1, i) for i in range(512)], np.uint64)
    c = np.array([oracle.ctr_draw(7, 1, 0, i) for i in range(512)], np.uint64)
    for other in (b, c):
        agree = np.unpackbits((~(a ^ other)).view(np.uint8)).mean()
        assert abs(agree - 0.5) < 5 * 0.5 / np.sqrt(512 * 64)


def test_oracle_counter_steps(oracle):
    X = Y = 256
    L = OracleLattice.flat(oracle, X, Y, 5)
    st0 = L.states.copy()
    p, q = oracle.resolve(0.5), oracle.resolve(0.0)
    L.step_ctr(oracle, p, q, 5, 50)
    assert L.t == 50 and L.phase == 0
    assert np.array_equal(L.states, st0)  # the xoshiro streams are not consumed
    h, err = oracle.reconstruct(L.planes)
    assert err is None  # curl-free, rows and columns close
    assert h.std() > 1.0  # KPZ growth roughens the flat start
    # deterministic in the seed, different across seeds
    L2 = OracleLattice.flat(oracle, X, Y, 5)
    L2.step_ctr(oracle, p, q, 5, 50)
    assert np.array_equal(L.planes, L2.planes)
    L3 = OracleLattice.flat(oracle, X, Y, 5)
    L3.step_ctr(oracle, p, q, 6, 50)
    assert not np.array_equal(L.planes, L3.planes)
