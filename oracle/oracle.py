"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (octoracle.c).
* ``RefLib``  -> oracle/_ref/libocref.so, the unmodified reference compiled
  from /root/reference/proj (absent unless built; see oracle/Makefile).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product package
(paper_1606_00310_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libocref.so")

ZERO, HALF, DYADIC, ARBITRARY = 0, 1, 2, 3
MODE_NAMES = {ZERO: "zero", HALF: "half", DYADIC: "dyadic", ARBITRARY: "arbitrary"}

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OOProb(C.Structure):
    _fields_ = [("r", C.c_double), ("mode", C.c_int), ("k", C.c_uint32), ("m", C.c_uint64)]


def _i128(lo: int, hi: int) -> int:
    v = (hi << 64) | lo
    return v - (1 << 128) if v >> 127 else v


class Oracle:
    """The C restatement. Field storage follows the reference SlopeField."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        L = self.L = C.CDLL(path)
        u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
        P = C.POINTER
        L.oo_rng_from_seed.argtypes = [u64, _u64p]
        L.oo_rng_next.argtypes = [_u64p]
        L.oo_rng_next.restype = u64
        L.oo_rng_jump.argtypes = [_u64p]
        L.oo_stream_set.argtypes = [u64, u32, _u64p]
        L.oo_dyadic_plan.argtypes = [C.c_double, u32, P(u32), P(u64)]
        L.oo_resolve.argtypes = [C.c_double, i32, P(OOProb)]
        L.oo_draws_per_word.argtypes = [P(OOProb), u32]
        L.oo_draws_per_word.restype = u32
        L.oo_xi_word.argtypes = [_u64p, P(OOProb), u32]
        L.oo_xi_word.restype = u64
        L.oo_new_flat.argtypes = [u32, u32, u32, _u64p]
        L.oo_sweep.argtypes = [u32, u32, u32, _u64p, _u64p, P(i32), i32, P(OOProb), P(OOProb), C.c_void_p]
        L.oo_step.argtypes = [u32, u32, u32, _u64p, _u64p, P(i32), P(u64), P(OOProb), P(OOProb), u64]
        L.oo_sweep_stripe.argtypes = [u32, u32, u32, u32, u32, _u64p, _u64p, _u64p, i32, P(OOProb), P(OOProb)]
        L.oo_field_checksum.argtypes = [u32, u32, u32, _u64p, u64]
        L.oo_field_checksum.restype = u64
        L.oo_states_digest.argtypes = [_u64p, u32]
        L.oo_states_digest.restype = u64
        L.oo_curl_check.argtypes = [u32, u32, u32, _u64p, P(u32), P(u32)]
        L.oo_curl_check.restype = u64
        L.oo_reconstruct.argtypes = [u32, u32, u32, _u64p, _i32p, P(i32), P(u32)]
        L.oo_power_sums.argtypes = [u32, u32, _i32p, _u64p]
        L.oo_measure_planes_mt.argtypes = [u32, u32, u32, _u64p, _u64p, P(i32), P(u64), P(u64)]
        L.oo_height_moments.argtypes = [u32, u32, _i32p, _f64p]
        L.oo_log_schedule.argtypes = [u64, u32, _u64p, u32]
        L.oo_log_schedule.restype = u32
        L.oo_mcs_stripe.argtypes = [u32, u32, u32, u32, u32, _u64p, _u64p, i32, P(OOProb), P(OOProb)]
        L.oo_ctr_draw.argtypes = [u64, u64, u32, u64]
        L.oo_ctr_draw.restype = u64
        L.oo_step_ctr.argtypes = [u32, u32, u32, _u64p, P(i32), P(u64), P(OOProb), P(OOProb), u64, u64]

    # -- opt-in counter-based streams (include/octgpu.h octgpu_set_rng) ---
    def ctr_draw(self, seed: int, sigma: int, y: int, i: int) -> int:
        return int(self.L.oo_ctr_draw(seed, sigma, y, i))

    # -- rng -------------------------------------------------------------
    def from_seed(self, seed: int) -> np.ndarray:
        st = np.zeros(4, np.uint64)
        self.L.oo_rng_from_seed(seed, st)
        return st

    def next(self, st: np.ndarray, n: int = 1) -> np.ndarray:
        return np.array([self.L.oo_rng_next(st) for _ in range(n)], np.uint64)

    def jump(self, st: np.ndarray) -> None:
        self.L.oo_rng_jump(st)

    def stream_set(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros((n, 4), np.uint64)
        self.L.oo_stream_set(seed, n, out)
        return out

    # -- params ----------------------------------------------------------
    def dyadic_plan(self, r: float, max_words: int = 16):
        k, m = C.c_uint32(), C.c_uint64()
        ok = self.L.oo_dyadic_plan(r, max_words, C.byref(k), C.byref(m))
        return (k.value, m.value) if ok else None

    def resolve(self, r: float, forced: int = -1) -> OOProb:
        p = OOProb()
        if self.L.oo_resolve(r, forced, C.byref(p)):
            raise ValueError(f"ConfigError: probability {r} / forced mode {forced}")
        return p

    def draws_per_word(self, p: OOProb, w: int = 64) -> int:
        return self.L.oo_draws_per_word(C.byref(p), w)

    def xi_words(self, st: np.ndarray, p: OOProb, w: int, n: int) -> np.ndarray:
        return np.array([self.L.oo_xi_word(st, C.byref(p), w) for _ in range(n)], np.uint64)

    # -- field -----------------------------------------------------------
    def new_flat(self, X: int, Y: int, w: int = 64) -> np.ndarray:
        planes = np.zeros((4, Y, X // (2 * w)), np.uint64)
        self.L.oo_new_flat(X, Y, w, planes)
        return planes

    def checksum(self, planes: np.ndarray, t: int, w: int = 64) -> int:
        _, Y, n = planes.shape
        return int(self.L.oo_field_checksum(n * 2 * w, Y, w, np.ascontiguousarray(planes), t))

    def states_digest(self, states: np.ndarray) -> int:
        return int(self.L.oo_states_digest(np.ascontiguousarray(states), states.shape[0]))

    def curl_check(self, planes: np.ndarray, w: int = 64):
        _, Y, n = planes.shape
        fx, fy = C.c_uint32(), C.c_uint32()
        bad = self.L.oo_curl_check(n * 2 * w, Y, w, np.ascontiguousarray(planes), C.byref(fx), C.byref(fy))
        return int(bad), (fx.value, fy.value)

    def reconstruct(self, planes: np.ndarray, w: int = 64):
        """Returns (heights, None) or (None, (kind, where)); kind 1 curl, 2 row0, 3 column."""
        _, Y, n = planes.shape
        X = n * 2 * w
        h = np.zeros((Y, X), np.int32)
        kind, where = C.c_int(), C.c_uint32()
        rc = self.L.oo_reconstruct(X, Y, w, np.ascontiguousarray(planes), h, C.byref(kind), C.byref(where))
        return (h, None) if rc == 0 else (None, (kind.value, where.value))

    def power_sums(self, h: np.ndarray) -> list[int]:
        Y, X = h.shape
        out = np.zeros(8, np.uint64)
        self.L.oo_power_sums(X, Y, np.ascontiguousarray(h, np.int32), out)
        return [_i128(int(out[2 * k]), int(out[2 * k + 1])) for k in range(4)]

    def measure_planes(self, planes: np.ndarray, w: int = 64):
        """reconstruct_heights + exact power sums straight from reference-layout planes (OpenMP, no
        HeightMap; for lattices of 2^32+ sites). Returns ([S1..S4], None) or (None, (kind, where, count))."""
        _, Y, n = planes.shape
        X = n * 2 * w
        out = np.zeros(8, np.uint64)
        kind, where, count = C.c_int(), C.c_uint64(), C.c_uint64()
        p = planes if (planes.dtype == np.uint64 and planes.flags.c_contiguous) else np.ascontiguousarray(planes, np.uint64)
        rc = self.L.oo_measure_planes_mt(X, Y, w, p, out, C.byref(kind), C.byref(where), C.byref(count))
        if rc:
            return None, (kind.value, where.value, count.value)
        return [_i128(int(out[2 * k]), int(out[2 * k + 1])) for k in range(4)], None

    def height_moments(self, h: np.ndarray) -> np.ndarray:
        Y, X = h.shape
        out = np.zeros(6, np.float64)
        self.L.oo_height_moments(X, Y, np.ascontiguousarray(h, np.int32), out)
        return out

    def log_schedule(self, t_max: int, ppd: int) -> list[int]:
        buf = np.zeros(4096, np.uint64)
        n = self.L.oo_log_schedule(t_max, ppd, buf, len(buf))
        return [int(v) for v in buf[:n]]


@dataclass
class OracleLattice:
    """Mutable lattice state driven by the C oracle (mirrors VecEngine)."""

    X: int
    Y: int
    w: int
    planes: np.ndarray
    states: np.ndarray
    t: int = 0
    phase: int = 0

    @classmethod
    def flat(cls, o: Oracle, X: int, Y: int, seed: int, w: int = 64) -> "OracleLattice":
        return cls(X, Y, w, o.new_flat(X, Y, w), o.stream_set(seed, Y))

    def step(self, o: Oracle, p: OOProb, q: OOProb, n: int = 1) -> None:
        ph, t = C.c_int(self.phase), C.c_uint64(self.t)
        o.L.oo_step(self.X, self.Y, self.w, self.planes, self.states, C.byref(ph), C.byref(t),
                    C.byref(p), C.byref(q), n)
        self.phase, self.t = ph.value, t.value

    def step_ctr(self, o: Oracle, p: OOProb, q: OOProb, seed: int, n: int = 1) -> None:
        """n MCS with the counter-based streams (states untouched)."""
        ph, t = C.c_int(self.phase), C.c_uint64(self.t)
        o.L.oo_step_ctr(self.X, self.Y, self.w, self.planes, C.byref(ph), C.byref(t), C.byref(p), C.byref(q),
                        seed, n)
        self.phase, self.t = ph.value, t.value

    def sweep(self, o: Oracle, parity: int, p: OOProb, q: OOProb, mask_log: np.ndarray | None = None) -> None:
        ph = C.c_int(self.phase)
        ml = mask_log.ctypes.data_as(C.c_void_p) if mask_log is not None else None
        rc = o.L.oo_sweep(self.X, self.Y, self.w, self.planes, self.states, C.byref(ph), parity,
                          C.byref(p), C.byref(q), ml)
        if rc:
            raise RuntimeError("InvariantError: sweep parity does not match field phase")
        self.phase = ph.value

    def checksum(self, o: Oracle) -> int:
        return o.checksum(self.planes, self.t, self.w)


class RefLib:
    """The unmodified reference, compiled into oracle/_ref/libocref.so."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference; run `make -C oracle`)")
        L = self.L = C.CDLL(path)
        u32, u64, i32, dbl, vp = C.c_uint32, C.c_uint64, C.c_int, C.c_double, C.c_void_p
        P = C.POINTER
        L.ocref_last_error.restype = C.c_char_p
        L.ocref_create.argtypes = [u32, u32, u32, u64, u32, i32, P(vp)]
        L.ocref_create_from.argtypes = [u32, u32, u32, u64, i32, _u64p, _u64p, u32, u64, u32, P(vp)]
        L.ocref_destroy.argtypes = [vp]
        L.ocref_step.argtypes = [vp, dbl, dbl, i32, i32, u64]
        L.ocref_sweep.argtypes = [vp, i32, dbl, dbl, i32, i32, vp]
        L.ocref_t.argtypes = [vp]
        L.ocref_t.restype = u64
        L.ocref_phase.argtypes = [vp]
        L.ocref_planes.argtypes = [vp, _u64p]
        L.ocref_states.argtypes = [vp, _u64p]
        L.ocref_checksum.argtypes = [vp]
        L.ocref_checksum.restype = u64
        L.ocref_heights.argtypes = [vp, _i32p]
        L.ocref_balances.argtypes = [vp, vp, vp]
        L.ocref_measure.argtypes = [vp, _f64p]
        L.ocref_height_moments.argtypes = [u32, u32, _i32p, _f64p]
        L.ocref_run.argtypes = [vp, dbl, dbl, i32, i32, u64, u32, _f64p, u32, P(u32)]
        L.ocref_log_schedule.argtypes = [u64, u32, _u64p, u32]
        L.ocref_log_schedule.restype = u32
        L.ocref_resolve.argtypes = [dbl, i32, u32, P(i32), P(u32), P(u32), P(u64)]
        L.ocref_rng_from_seed.argtypes = [u64, _u64p]
        L.ocref_rng_next.argtypes = [_u64p, _u64p, u32]
        L.ocref_rng_jump.argtypes = [_u64p]
        L.ocref_stream_set.argtypes = [u64, u32, _u64p]
        L.ocref_xi_words.argtypes = [_u64p, dbl, i32, u32, _u64p, u32]
        L.ocref_curl_check.argtypes = [u32, u32, u32, _u64p, P(u64), P(u32), P(u32)]
        L.ocref_reconstruct.argtypes = [u32, u32, u32, _u64p, _i32p]
        L.ocref_snapshot.argtypes = [vp, C.c_char_p, C.c_int64]
        L.ocref_snapshot.restype = C.c_int64
        L.ocref_run_session.argtypes = [u32, u32, u32, dbl, dbl, u64, u32, u64, u32, C.c_char_p, C.c_char_p,
                                        C.c_char_p]

    def err(self) -> str:
        return self.L.ocref_last_error().decode()

    def check(self, rc: int) -> None:
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.err()}")


class RefEngine:
    """Handle to a reference VecEngine (kind 0) or RefEngine (kind 1)."""

    def __init__(self, lib: RefLib, X: int, Y: int, seed: int, w: int = 64, workers: int = 1, kind: int = 0,
                 _handle=None):
        self.lib, self.X, self.Y, self.w = lib, X, Y, w
        self.n = X // (2 * w)
        if _handle is not None:
            self.h = _handle
        else:
            h = C.c_void_p()
            lib.check(lib.L.ocref_create(X, Y, w, seed, workers, kind, C.byref(h)))
            self.h = h

    @classmethod
    def from_state(cls, lib: RefLib, X, Y, w, t, phase, planes, states, master_seed=0, workers=1):
        h = C.c_void_p()
        st = np.ascontiguousarray(states, np.uint64)
        lib.check(lib.L.ocref_create_from(X, Y, w, t, phase, np.ascontiguousarray(planes, np.uint64), st,
                                          st.shape[0], master_seed, workers, C.byref(h)))
        return cls(lib, X, Y, 0, w, workers, 0, _handle=h)

    def __del__(self):
        try:
            self.lib.L.ocref_destroy(self.h)
        except Exception:
            pass

    def step(self, p: float, q: float, n: int = 1, pmode: int = -1, qmode: int = -1) -> None:
        self.lib.check(self.lib.L.ocref_step(self.h, p, q, pmode, qmode, n))

    def sweep(self, parity: int, p: float, q: float, pmode=-1, qmode=-1, mask_log: np.ndarray | None = None):
        ml = mask_log.ctypes.data_as(C.c_void_p) if mask_log is not None else None
        self.lib.check(self.lib.L.ocref_sweep(self.h, parity, p, q, pmode, qmode, ml))

    @property
    def t(self) -> int:
        return int(self.lib.L.ocref_t(self.h))

    @property
    def phase(self) -> int:
        return int(self.lib.L.ocref_phase(self.h))

    def planes(self) -> np.ndarray:
        out = np.zeros((4, self.Y, self.n), np.uint64)
        self.lib.L.ocref_planes(self.h, out)
        return out

    def states(self) -> np.ndarray:
        out = np.zeros((self.Y, 4), np.uint64)
        self.lib.L.ocref_states(self.h, out)
        return out

    def checksum(self) -> int:
        return int(self.lib.L.ocref_checksum(self.h))

    def heights(self) -> np.ndarray:
        out = np.zeros((self.Y, self.X), np.int32)
        self.lib.check(self.lib.L.ocref_heights(self.h, out))
        return out

    def balances(self) -> tuple[np.ndarray, np.ndarray]:
        """(row_balances, col_balances) of the reference field (slope_field.hpp:177-202)."""
        rows, cols = np.zeros(self.Y, np.int64), np.zeros(self.X, np.int64)
        self.lib.L.ocref_balances(self.h, rows.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p))
        return rows, cols

    def measure(self) -> np.ndarray:
        out = np.zeros(4, np.float64)
        self.lib.check(self.lib.L.ocref_measure(self.h, out))
        return out

    def run(self, p, q, tmax, ppd, pmode=-1, qmode=-1) -> np.ndarray:
        out = np.zeros((4096, 5), np.float64)
        n = C.c_uint32()
        self.lib.check(self.lib.L.ocref_run(self.h, p, q, pmode, qmode, tmax, ppd, out, 4096, C.byref(n)))
        return out[: n.value].copy()

    def snapshot(self) -> bytes:
        size = self.lib.L.ocref_snapshot(self.h, None, 0)
        buf = C.create_string_buffer(size)
        self.lib.L.ocref_snapshot(self.h, buf, size)
        return buf.raw


class OracleStripe:
    """CPU stand-in for paper_1606_00310_b200.stripes.StripeEngine (test infra):
    same pack/unpack/mcs/finish/measure_local contract and buffer layout
    (5 halo rows above, 6 below: engine.cu kStripeHA / kStripeHB), computed by
    oo_mcs_stripe (the reference's sweeps restricted to a stripe with halos)."""

    HA, HB = 5, 6

    def __init__(self, o: Oracle, X: int, Y: int, y0: int, y1: int, seed: int, w: int = 64):
        self.o, self.X, self.Y, self.w, self.y0, self.y1 = o, X, Y, w, y0, y1
        self.L = L = y1 - y0
        self.n = n = X // (2 * w)
        HA, HB = self.HA, self.HB
        full = o.new_flat(X, Y, w)
        self.buf = np.zeros((4, HA + L + HB, n), np.uint64)
        self.buf[:, HA:HA + L] = full[:, y0:y1]
        self.st = np.zeros((HA + L + HB, 4), np.uint64)
        self.st[HA:HA + L] = o.stream_set(seed, y1)[y0:y1]
        self.t, self.phase = 0, 0
        self.to_prev_bytes = HB * (4 * n + 4) * 8
        self.to_next_bytes = HA * (4 * n + 4) * 8
        self.boundary_bytes = n * 8

    @staticmethod
    def _u64(t):
        return t.numpy().view(np.uint64)

    def _gather(self, r0, nrows, out):
        a = self._u64(out)
        k = 4 * nrows * self.n
        a[:k] = self.buf[:, r0:r0 + nrows].ravel()
        a[k:] = self.st[r0:r0 + nrows].ravel()

    def _scatter(self, r0, nrows, src):
        a = self._u64(src)
        k = 4 * nrows * self.n
        self.buf[:, r0:r0 + nrows] = a[:k].reshape(4, nrows, self.n)
        self.st[r0:r0 + nrows] = a[k:].reshape(nrows, 4)

    def pack(self, to_prev, to_next):
        self._gather(self.HA, self.HB, to_prev)
        self._gather(self.L, self.HA, to_next)

    def unpack(self, from_prev, from_next):
        self._scatter(0, self.HA, from_prev)
        self._scatter(self.HA + self.L, self.HB, from_next)

    def max_mcs(self, prm):
        return 3  # the CPU stand-in runs the 3-MCS protocol for every mode

    def mcs(self, prm, boundary_out, n=1):
        o = self.o
        p = o.resolve(prm.p.value, int(prm.p.mode))
        q = o.resolve(prm.q.value, int(prm.q.mode))
        yoff = (self.y0 - self.HA) % self.Y
        R = self.HA + self.L + self.HB
        o.L.oo_mcs_stripe(self.X, self.w, R, 2 * n, yoff, self.buf, self.st, self.phase, C.byref(p), C.byref(q))
        self._u64(boundary_out)[:] = self.buf[2 + self.phase, self.HA + self.L]
        self.t += n

    def finish(self, boundary_in):
        self.buf[2 + self.phase, self.HA] = self._u64(boundary_in)

    def planes(self):
        return self.buf[:, self.HA:self.HA + self.L].copy()

    def states(self):
        return self.st[self.HA:self.HA + self.L].copy()

    def measure_local(self):
        """Stripe-local power sums in the GPU kernels' gauge (numpy, no curl check)."""
        from paper_1606_00310_b200.stripes import StripeMoments

        X, L = self.X, self.L
        bits = lambda words: np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")  # noqa
        S = [0, 0, 0, 0]
        G = 0
        col = 0
        sy_first = row_first = None
        for l in range(1, L + 1):
            y = (self.y0 + l - 1) % self.Y
            r = self.HA + l - 1
            a = bits(self.buf[y & 1, r]).astype(np.int64)
            b = bits(self.buf[(y & 1) ^ 1, r]).astype(np.int64)
            sig = np.empty(X, np.int64)
            sig[0::2], sig[1::2] = 2 * a - 1, 2 * b - 1
            sy = 1 if int(self.buf[2 + (y & 1), r, 0]) & 1 else -1
            G += sy
            col += sy
            if l == 1:
                sy_first, row_first = sy, int(sig.sum())
            h = (G - int(sig[0])) + np.cumsum(sig)
            for k in range(4):
                S[k] += int(np.sum(h.astype(object) ** (k + 1)))
        return StripeMoments(self.y0, self.t, X * L, tuple(S), col, sy_first, row_first, 0, -1)
