"""GpuEngine — the B200 drop-in for ``octsca::VecEngine<Word>`` (engine_vec.hpp:184-213).

Same facade: construct from (LatticeConfig, seed) or from (SlopeField,
RngStreamSet); ``step(prm)``, ``t``, ``field()``, ``streams()``,
``heights()``, plus ``measure()`` (device-side W² without a HeightMap) and
``sweep()`` (``sublattice_sweep`` with optional mask log). All state lives on
the GPU; ``field()``/``streams()``/``heights()`` copy to the host on demand.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from ._lib import ConfigError, OctMoments, check, lib
from .params import LatticeConfig, UpdateParams


def _word_dtype(w: int):
    return np.uint64 if w == 64 else np.uint32


@dataclass
class SlopeField:
    """Host copy of the bit planes in the reference layout (slope_field.hpp:22-102).

    planes: (4, Y, n) array, plane order x/even, x/odd, y/even, y/odd."""

    cfg: LatticeConfig
    planes: np.ndarray
    t_mcs: int = 0
    phase: int = 0

    @staticmethod
    def plane_index(axis: int, parity: int) -> int:
        return axis * 2 + parity

    def row(self, axis: int, parity: int, y: int) -> np.ndarray:
        return self.planes[self.plane_index(axis, parity), y]

    def minus_bit(self, axis: int, x: int, y: int) -> int:
        par = (x ^ y) & 1
        j = x >> 1
        w = self.cfg.w
        return int((int(self.planes[axis * 2 + par, y, j // w]) >> (j % w)) & 1)

    def __eq__(self, o: object) -> bool:
        return (isinstance(o, SlopeField) and self.cfg == o.cfg and self.t_mcs == o.t_mcs
                and self.phase == o.phase and np.array_equal(self.planes, o.planes))


def new_flat(cfg: LatticeConfig) -> SlopeField:
    """slope_field.hpp:110-118 (host copy, e.g. for create_from)."""
    cfg.validate()
    dt = _word_dtype(cfg.w)
    planes = np.zeros((4, cfg.Y, cfg.words_per_row()), dt)
    planes[1] = np.iinfo(dt).max
    planes[3] = np.iinfo(dt).max
    return SlopeField(cfg, planes)


@dataclass
class RngStreamSet:
    """rng.hpp:80-120: one xoshiro256++ state per row, (n, 4) uint64."""

    master_seed: int
    states: np.ndarray

    @staticmethod
    def derive(master_seed: int, n: int) -> "RngStreamSet":
        out = np.zeros((n, 4), np.uint64)
        check(lib().octgpu_stream_states(master_seed, n, out.ctypes.data_as(C.c_void_p)))
        return RngStreamSet(master_seed, out)

    def size(self) -> int:
        return int(self.states.shape[0])


@dataclass
class HeightMap:
    """lattice.hpp:53-107: h[y, x] int32, mean."""

    X: int
    Y: int
    h: np.ndarray
    mean: float = 0.0


@dataclass
class MeasurementRecord:
    """measure.hpp:11-17, plus the exact integer statistics it derives from."""

    t: int
    W2: float
    mean_h: float
    skew: float
    kurt: float
    n_sites: int = 0
    power_sums: tuple = field(default_factory=tuple)  # (S1, S2, S3, S4), exact ints, gauge h(0,0)=0

    def W2_exact(self) -> Fraction:
        N = self.n_sites
        S1, S2 = self.power_sums[0], self.power_sums[1]
        return Fraction(N * S2 - S1 * S1, N * N)

    def mean_exact(self) -> Fraction:
        return Fraction(self.power_sums[0], self.n_sites)


def field_checksum(f: SlopeField) -> int:
    """slope_field.hpp:232-246 (FNV-1a over the 4 planes, then t_mcs)."""
    h = 0xCBF29CE484222325
    data = np.ascontiguousarray(f.planes).astype(np.uint64).tobytes()
    # little-endian u64 bytes of every word, then t_mcs
    for b in data + int(f.t_mcs).to_bytes(8, "little"):
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _i128(lo: int, hi: int) -> int:
    v = ((hi & 0xFFFFFFFFFFFFFFFF) << 64) | lo
    return v - (1 << 128) if v >> 127 else v


def release_pool(device: int = 0) -> None:
    """Return the unused memory of the library's plane-set pool on `device` to the driver
    (octgpu_release_pool): periodic engines keep freed plane sets for the next engine of the process."""
    check(lib().octgpu_release_pool(device))


class GpuEngine:
    """Drop-in for ``VecEngine<Word>``; ``workers`` is accepted and ignored
    (the GPU partition is fixed and results are partition-independent, as the
    reference's are across worker counts, engine_vec.hpp:141-144)."""

    def __init__(self, cfg: LatticeConfig | SlopeField, seed: int | RngStreamSet = 1, workers: int = 1,
                 device: int = 0):
        self._h = None
        L = lib()
        h = C.c_void_p()
        if isinstance(cfg, SlopeField):
            f, streams = cfg, seed
            if not isinstance(streams, RngStreamSet):
                raise TypeError("GpuEngine(SlopeField, RngStreamSet, workers)")
            c = f.cfg
            planes = np.ascontiguousarray(f.planes, _word_dtype(c.w))
            st = np.ascontiguousarray(streams.states, np.uint64)
            check(L.octgpu_create_from(c.X, c.Y, c.w, int(f.t_mcs), int(f.phase),
                                       planes.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p),
                                       st.shape[0], int(streams.master_seed), device, C.byref(h)))
            self.cfg = c
        else:
            check(L.octgpu_create(cfg.X, cfg.Y, cfg.w, int(seed), device, C.byref(h)))
            self.cfg = cfg
        self._h = h
        self.device = device

    name = "gpu"

    def __del__(self, _lib=lib):  # the module global may already be gone at interpreter shutdown
        if getattr(self, "_h", None):
            _lib().octgpu_destroy(self._h)
            self._h = None

    def close(self) -> None:
        self.__del__()

    # -- hot path ------------------------------------------------------------
    def step(self, prm: UpdateParams, n: int = 1) -> None:
        """n x VecEngine::step (engine_vec.hpp:197)."""
        c = prm.to_c()
        check(lib().octgpu_step(self._h, C.byref(c), int(n)))

    def sweep(self, parity: int, prm: UpdateParams, mask_log: bool = False):
        """sublattice_sweep (engine_vec.hpp:145-168); returns the (Y, n) mask log if asked."""
        c = prm.to_c()
        buf = None
        if mask_log:
            buf = np.zeros((self.cfg.Y, self.cfg.words_per_row()), _word_dtype(self.cfg.w))
        check(lib().octgpu_sweep(self._h, int(parity), C.byref(c),
                                 buf.ctypes.data_as(C.c_void_p) if buf is not None else None))
        return buf

    def set_tile_shift(self, seed: int) -> None:
        """Random per-pass row origin of the kernels' block tiling (DTr-style); 0 = off. Result-neutral."""
        check(lib().octgpu_set_tile_shift(self._h, int(seed)))

    RNG_KINDS = {"xoshiro": 0, "counter": 1}

    def set_rng(self, kind: str) -> None:
        """xi source of step(): "xoshiro" (default; the reference's per-row streams, bit-exact) or
        "counter" (opt-in counter-based SplitMix64 streams keyed by (master seed, sweep, row); no
        reference equivalent, pinned by the oracle's oo_step_ctr). See include/octgpu.h."""
        if kind not in self.RNG_KINDS:
            raise ValueError(f"rng kind must be one of {sorted(self.RNG_KINDS)}")
        check(lib().octgpu_set_rng(self._h, self.RNG_KINDS[kind]))

    @property
    def rng(self) -> str:
        k = int(lib().octgpu_get_rng(self._h))
        return {v: n for n, v in self.RNG_KINDS.items()}[k]

    KERNELS = {0: "k_mcs", 1: "k_mcs_bulk", 2: "k_mcs_deep", 3: "k_sweep_ctr"}

    def pass_plan(self, prm: UpdateParams) -> tuple[str, float]:
        """(kernel, MCS per launch) of the passes step(prm) launches on this engine (octgpu_pass_plan)."""
        c = prm.to_c()
        k, sw = C.c_int(), C.c_int()
        check(lib().octgpu_pass_plan(self._h, C.byref(c), C.byref(k), C.byref(sw)))
        return self.KERNELS[k.value], sw.value / 2

    def set_stream(self, cuda_stream: int | None) -> None:
        check(lib().octgpu_set_stream(self._h, C.c_void_p(cuda_stream) if cuda_stream else None))

    def sync(self) -> None:
        check(lib().octgpu_sync(self._h))

    # -- state -----------------------------------------------------------------
    @property
    def t(self) -> int:
        return int(lib().octgpu_t(self._h))

    @property
    def phase(self) -> int:
        return int(lib().octgpu_phase(self._h))

    @property
    def launches(self) -> int:
        return int(lib().octgpu_launch_count(self._h))

    def planes(self, out: np.ndarray | None = None) -> np.ndarray:
        """The four bit-planes in the reference layout [4][Y][n]; `out` (e.g. a
        pinned buffer) is filled in place when given."""
        c = self.cfg
        shape, dt = (4, c.Y, c.words_per_row()), _word_dtype(c.w)
        if out is None:
            out = np.zeros(shape, dt)
        elif out.shape != shape or out.dtype != dt or not out.flags.c_contiguous:
            raise ConfigError(f"planes buffer must be a C-contiguous {dt.__name__} array of shape {shape}")
        check(lib().octgpu_get_planes(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def field(self) -> SlopeField:
        return SlopeField(self.cfg, self.planes(), self.t, self.phase)

    slope_field = field

    def streams(self, out: np.ndarray | None = None) -> RngStreamSet:
        if out is None:
            out = np.zeros((self.cfg.Y, 4), np.uint64)
        elif out.shape != (self.cfg.Y, 4) or out.dtype != np.uint64 or not out.flags.c_contiguous:
            raise ConfigError(f"states buffer must be a C-contiguous uint64 array of shape ({self.cfg.Y}, 4)")
        check(lib().octgpu_get_states(self._h, out.ctypes.data_as(C.c_void_p)))
        return RngStreamSet(int(lib().octgpu_master_seed(self._h)), out)

    def checksum(self) -> int:
        v = C.c_uint64()
        check(lib().octgpu_field_checksum(self._h, C.byref(v)))
        return int(v.value)

    # -- measurement ---------------------------------------------------------
    def heights(self) -> HeightMap:
        """reconstruct_heights(field) (slope_field.hpp:206-229) on the device."""
        c = self.cfg
        out = np.zeros((c.Y, c.X), np.int32)
        check(lib().octgpu_heights(self._h, out.ctypes.data_as(C.c_void_p)))
        return HeightMap(c.X, c.Y, out, float(out.mean(dtype=np.float64)))

    def row_balances(self) -> np.ndarray:
        """row_balances(field) (slope_field.hpp:177-189): sum_x sigma_x-(x, y) per row, on the device."""
        out = np.zeros(self.cfg.Y, np.int64)
        check(lib().octgpu_balances(self._h, out.ctypes.data_as(C.c_void_p), None))
        return out

    def col_balances(self) -> np.ndarray:
        """col_balances(field) (slope_field.hpp:192-202): sum_y sigma_y-(x, y) per column, on the device."""
        out = np.zeros(self.cfg.X, np.int64)
        check(lib().octgpu_balances(self._h, None, out.ctypes.data_as(C.c_void_p)))
        return out

    def measure(self) -> MeasurementRecord:
        """measure_heights(t, heights()) without materialising heights."""
        m = OctMoments()
        check(lib().octgpu_measure(self._h, C.byref(m)))
        sums = tuple(_i128(int(m.s_lo[k]), int(m.s_hi[k])) for k in range(4))
        return MeasurementRecord(int(m.t), m.W2, m.mean_h, m.skew, m.kurt, int(m.n_sites), sums)
