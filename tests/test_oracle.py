"""Pin the CPU oracle (oracle/octoracle.c) to the reference.

(a) against the golden vectors generated from the unmodified reference
    (tests/golden/goldens.json, tests/golden/make_goldens.py) and SURVEY.md
    Appendix A; (b) against the reference itself (oracle/_ref) when built.
Also checks the algebraic facts the GPU path relies on (integer threshold,
dyadic exactness, word-parallel curl formula, jump-ahead linearity).
"""
import itertools
import math
import random

import numpy as np
import pytest

from oracle import ARBITRARY, DYADIC, OracleLattice, RefEngine

H = lambda v: int(v, 16)  # noqa: E731


def test_rng_kats(oracle, goldens):
    k = goldens["kat"]
    st = oracle.from_seed(1)
    assert [int(v) for v in st] == [H(v) for v in k["from_seed_1"]]
    assert [int(v) for v in oracle.next(st.copy(), 4)] == [H(v) for v in k["next4"]]
    ss = oracle.stream_set(1, 3)
    assert [[int(v) for v in r] for r in ss] == [[H(v) for v in r] for r in k["stream_set_1_3"]]
    j = oracle.from_seed(1)
    oracle.jump(j)
    assert [int(v) for v in j] == [H(v) for v in k["jump_from_seed_1"]]
    # SURVEY.md Appendix A
    assert [int(v) for v in oracle.from_seed(1)] == [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E,
                                                      0x71C18690EE42C90B]


def test_xi_words(oracle, goldens):
    for case in goldens["xi_words"]:
        p = oracle.resolve(case["r"], case["forced"])
        st = oracle.from_seed(case["seed"])
        words = oracle.xi_words(st, p, case["w"], 8)
        assert [int(v) for v in words] == [H(v) for v in case["words"]], case
        assert [int(v) for v in st] == [H(v) for v in case["state_after"]], case


def test_resolve(oracle, goldens):
    for case in goldens["resolve"]:
        if case["rc"]:
            with pytest.raises(ValueError):
                oracle.resolve(case["r"], case["forced"])
            continue
        p = oracle.resolve(case["r"], case["forced"])
        assert p.mode == case["mode"], case
        assert oracle.draws_per_word(p, 64) == case["draws"], case
        if p.mode == DYADIC:
            assert (p.k, p.m) == (case["k"], case["m"]), case


def test_dyadic_plans_appendix_a(oracle):
    assert oracle.dyadic_plan(0.75) == (2, 3)
    assert oracle.dyadic_plan(0.8125) == (4, 13)
    assert oracle.dyadic_plan(0.25) == (2, 1)
    assert oracle.dyadic_plan(0.375) == (3, 3)
    assert oracle.dyadic_plan(0.95) is None
    assert oracle.dyadic_plan(1.0) is None


@pytest.mark.parametrize("k", range(1, 9))
def test_dyadic_exact_bruteforce(oracle, k):
    """SPEC.md acceptance #8: every plan with k <= 8 realises m/2^k exactly.
    Horner AND/OR over k fair bits (rng.hpp:157-164), all 2^k inputs."""
    for m in range(1, 2 ** k, 2):
        r = m / 2 ** k
        kk, mm = oracle.dyadic_plan(r)
        assert (kk, mm) == (k, m)
        ones = 0
        for bits in itertools.product((0, 1), repeat=kk):
            acc = bits[0]
            for i in range(1, kk):
                acc = (acc | bits[i]) if (mm >> i) & 1 else (acc & bits[i])
            ones += acc
        assert ones == m


def test_integer_threshold_equals_to_unit():
    """to_unit(x) < r  <=>  (x >> 11) < ceil(r * 2^53)  (rng.hpp:167-177); the GPU uses the right side."""
    rs = [0.95, 0.98, 0.02, 1.0, 1 - 2 ** -53, 2 ** -53, 0.3, 0.1, 1 / 3, 0.999999, 5e-324, 0.7071067811865476]
    rnd = random.Random(5)
    for r in rs:
        thr = math.ceil(math.ldexp(r, 53))
        xs = [rnd.getrandbits(64) for _ in range(2000)]
        for t in (thr - 1, thr, thr + 1):
            if 0 <= t < 2 ** 53:
                xs += [t << 11, (t << 11) | 0x7FF]
        for x in xs:
            lhs = float(x >> 11) * 2.0 ** -53 < r
            assert lhs == ((x >> 11) < thr), (r, x)


def _curl_wordparallel(planes: np.ndarray) -> int:
    """Word-parallel curl check used by the measurement kernel."""
    _, Y, n = planes.shape
    bad = 0
    one = np.uint64(1)
    for y in range(Y):
        for pi in (0, 1):
            A = planes[pi, y]
            B = planes[pi ^ 1, (y - 1) % Y]
            C = planes[2 + pi, y]
            Dr = planes[2 + (pi ^ 1), y]
            if ((pi ^ y) & 1) == 0:  # sites at even x: sigma_y-(x-1) sits one packed bit lower
                D = (Dr << one) | (np.roll(Dr, 1) >> np.uint64(63))
            else:
                D = Dr
            V = (A ^ B ^ C ^ D) | ((A ^ B) & (A ^ C))
            bad += sum(bin(int(v)).count("1") for v in V)
    return bad


def test_curl_formula_matches_scalar(oracle):
    rnd = np.random.default_rng(3)
    L = OracleLattice.flat(oracle, 256, 16, 11)
    L.step(oracle, oracle.resolve(0.5), oracle.resolve(0.0), 30)
    assert oracle.curl_check(L.planes)[0] == 0 == _curl_wordparallel(L.planes)
    for trial in range(40):
        P = L.planes.copy()
        for _ in range(rnd.integers(1, 4)):
            pl, y, k, b = rnd.integers(4), rnd.integers(16), rnd.integers(2), rnd.integers(64)
            P[pl, y, k] ^= np.uint64(1) << np.uint64(b)
        assert oracle.curl_check(P)[0] == _curl_wordparallel(P), trial


def test_log_schedule(oracle, goldens):
    for key, val in goldens["log_schedule"].items():
        t, p = map(int, key.split(","))
        assert oracle.log_schedule(t, p) == val
    assert len(goldens["log_schedule"]["10000,8"]) == 33


def _power_sums(r):
    return [int(v) for v in r["power_sums"]]


@pytest.mark.parametrize("idx", range(25))
def test_oracle_runs_match_reference_goldens(oracle, goldens, idx):
    r = goldens["runs"][idx]
    if r["X"] * r["Y"] * r["mcs"] > 3e8 and oracle.resolve(r["p"]).mode == ARBITRARY:
        pytest.skip("slow in the scalar oracle; covered by the GPU parity suite")
    L = OracleLattice.flat(oracle, r["X"], r["Y"], r["seed"], r["w"])
    L.step(oracle, oracle.resolve(r["p"]), oracle.resolve(r["q"]), r["mcs"])
    assert hex(L.checksum(oracle)) == r["checksum"]
    assert hex(oracle.states_digest(L.states)) == r["states_digest"]
    h, err = oracle.reconstruct(L.planes, r["w"])
    assert err is None
    assert oracle.power_sums(h) == _power_sums(r)
    m = oracle.height_moments(h)
    assert m[0] == r["mean_h"] and m[1] == r["W2"]  # bit-exact sequential doubles


APPENDIX_A = {  # (p, q, seed) -> field_checksum after 1000 MCS at 1024^2
    (1.0, 0.0, 1): 0x41EE5A09BBC966DC, (0.5, 0.0, 1): 0xB482F51D70B20474, (0.5, 0.0, 42): 0xA600D78D6457EDEB,
    (0.5, 0.5, 1): 0x8AD7920A8251C44B, (0.75, 0.0, 1): 0x5A8FA41A05B8C63D,
}


def test_goldens_agree_with_survey_appendix_a(goldens):
    got = {(r["p"], r["q"], r["seed"]): H(r["checksum"]) for r in goldens["runs"] if r["X"] == 1024}
    for k, v in APPENDIX_A.items():
        assert got[k] == v
    s = goldens["sessions"][0]
    assert s["csv_sha256"] == "3dccb6ae8ccd29277a7550f595124698fac110a25ab1441e91c1eb45f1a5dccc"
    assert s["snap_sha256"] == "285cc28a64094f5378747aa2a5e297f467c4c848306bf468fdb275bd5d71e501"


# ---- direct cross-checks against the compiled reference (when built) ----

@pytest.mark.parametrize("p,q,X,Y,w,seed", [
    (0.5, 0.0, 256, 34, 64, 1), (0.75, 0.25, 384, 30, 64, 2), (0.95, 0.0, 128, 8, 64, 3),
    (0.98, 0.02, 256, 4, 64, 4), (1.0, 0.0, 128, 6, 64, 5), (0.5, 0.5, 128, 10, 32, 6), (0.0, 0.5, 192, 12, 32, 7),
])
def test_oracle_sweeps_match_reference(oracle, reflib, p, q, X, Y, w, seed):
    ref = RefEngine(reflib, X, Y, seed, w=w, workers=3)
    L = OracleLattice.flat(oracle, X, Y, seed, w)
    pp, qq = oracle.resolve(p), oracle.resolve(q)
    n = X // (2 * w)
    for parity in (0, 1, 0, 1, 0):
        log_o = np.zeros((Y, n), np.uint64)
        log_r = np.zeros((Y, n), np.uint64)
        L.sweep(oracle, parity, pp, qq, log_o)
        ref.sweep(parity, p, q, mask_log=log_r)
        assert np.array_equal(log_o, log_r)
        assert np.array_equal(L.planes, ref.planes())
        assert np.array_equal(L.states, ref.states())


def test_oracle_heights_match_reference(oracle, reflib):
    ref = RefEngine(reflib, 256, 32, 9, workers=2)
    ref.step(0.5, 0.25, 25)
    h_ref = ref.heights()
    h, err = oracle.reconstruct(ref.planes())
    assert err is None and np.array_equal(h, h_ref)
    m_ref = np.zeros(6)
    reflib.L.ocref_height_moments(256, 32, np.ascontiguousarray(h_ref), m_ref)
    assert np.array_equal(oracle.height_moments(h), m_ref)


def test_stripe_sweep_equals_full_sweep(oracle):
    """oo_sweep_stripe (used by the multi-rank tests) partitions exactly."""
    X, Y = 256, 12
    L = OracleLattice.flat(oracle, X, Y, 21)
    pp, qq = oracle.resolve(0.5), oracle.resolve(0.5)
    L.step(oracle, pp, qq, 3)
    full = L.planes.copy()
    st_full = L.states.copy()
    ph = L.phase
    L.sweep(oracle, ph, pp, qq)
    bounds = [(0, 4), (4, 10), (10, 12)]
    planes = full.copy()
    states = st_full.copy()
    outs = []
    for (y0, y1) in bounds:
        sp = np.ascontiguousarray(planes[:, y0:y1])
        ghost = planes[2 + (ph ^ 1), y1 % Y].copy()
        st = np.ascontiguousarray(states[y0:y1])
        oracle.L.oo_sweep_stripe(X, Y, 64, y0, y1, sp, ghost, st, ph, pp, qq)
        outs.append((y0, y1, sp, ghost, st))
    res = planes.copy()
    for (y0, y1, sp, ghost, st) in outs:
        res[:, y0:y1] = sp
    for (y0, y1, sp, ghost, st) in outs:  # write back the borrowed ghost rows (one owner each)
        res[2 + (ph ^ 1), y1 % Y] = ghost
    assert np.array_equal(res, L.planes)
    assert np.array_equal(np.concatenate([o[4] for o in outs]), L.states)


@pytest.mark.parametrize("r", [0.5, 0.75, 0.95])
def test_xi_bit_frequencies_4sigma(oracle, r):
    """SPEC.md acceptance 8: bit frequencies of the xi words at 4 sigma over 10^6 words
    (the oracle's xi words are pinned to the reference's by test_xi_words)."""
    import numpy as np

    nwords = 10 ** 6
    st = oracle.stream_set(2024, 1)[0].copy()
    words = oracle.xi_words(st, oracle.resolve(r), 64, nwords)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little").reshape(nwords, 64)
    per_pos = bits.mean(axis=0)
    sig_pos = (r * (1 - r) / nwords) ** 0.5
    assert np.all(np.abs(per_pos - r) <= 4 * sig_pos), per_pos
    assert abs(bits.mean() - r) <= 4 * sig_pos / 8


# ---------------------------------------------------------------------------
# the at-scale checker (oo_measure_planes_mt) against the scalar reconstruct + power sums, and the
# reference's own heights; balances against the reference

@pytest.mark.parametrize("geom", [(128, 2, 64), (256, 34, 64), (384, 62, 64), (192, 66, 32), (1024, 64, 64)])
def test_measure_planes_mt_equals_reconstruct(oracle, geom):
    X, Y, w = geom
    L = OracleLattice.flat(oracle, X, Y, 3 + X + Y, w)
    L.step(oracle, oracle.resolve(0.5), oracle.resolve(0.25), 9)
    h, err = oracle.reconstruct(L.planes, w)
    assert err is None
    sums, err = oracle.measure_planes(L.planes, w)
    assert err is None
    assert sums == oracle.power_sums(h)


def test_measure_planes_mt_reports_reconstruct_errors(oracle):
    X, Y = 256, 34
    L = OracleLattice.flat(oracle, X, Y, 5)
    L.step(oracle, oracle.resolve(0.75), oracle.resolve(0.0), 4)
    bad = L.planes.copy()
    bad[2, 7, 1] ^= np.uint64(1 << 5)  # one y-slope flipped: curl violations
    n_bad, (fx, fy) = oracle.curl_check(bad)
    sums, err = oracle.measure_planes(bad)
    assert sums is None and err[0] == 1 and err[2] == n_bad and err[1] == fy * X + fx
    # a uniform tilt (every slope +1) is curl-free but breaks the row-0 closure
    tilt = np.full((4, Y, X // 128), ~np.uint64(0), np.uint64)
    assert oracle.measure_planes(tilt)[1][0] == 2
    _, e2 = oracle.reconstruct(tilt)
    assert e2[0] == 2


def test_balances_reference_on_random_field(oracle, reflib):
    X, Y = 256, 34
    ref = RefEngine(reflib, X, Y, 11, workers=2)
    ref.step(0.5, 0.25, 7)
    rows, cols = ref.balances()
    assert rows.shape == (Y,) and cols.shape == (X,)
    assert not rows.any() and not cols.any()  # a valid periodic surface
    # a broken field: the reference's balances are what the GPU export must reproduce (test_parity_gpu)
    planes = ref.planes()
    planes[2, 3, 0] ^= np.uint64(0b101)
    planes[0, 5, 1] ^= np.uint64(1 << 9)
    bad = RefEngine.from_state(reflib, X, Y, 64, 7, 0, planes, ref.states())
    r2, c2 = bad.balances()
    assert r2[5] != 0 and (c2 != 0).sum() == 2
