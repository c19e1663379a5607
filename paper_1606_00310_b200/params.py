"""Lattice geometry and update parameters, mirroring the reference types.

* ``LatticeConfig``  <- octsca::LatticeConfig (lattice.hpp:26-48)
* ``ProbMode``       <- octsca::ProbMode (params.hpp:13)
* ``ProbSpec``       <- octsca::ProbSpec (params.hpp:28-81); resolution runs in
  liboctgpu (``octgpu_resolve``), the same code the engine uses.
* ``UpdateParams``   <- octsca::UpdateParams (params.hpp:95-102)
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

from ._lib import OctParams, OctProb, check, lib


class ProbMode(enum.IntEnum):
    Zero = 0
    Half = 1
    Dyadic = 2
    Arbitrary = 3

    @property
    def label(self) -> str:  # prob_mode_name (params.hpp:15-26)
        return self.name.lower()


@dataclass(frozen=True)
class LatticeConfig:
    X: int
    Y: int
    w: int = 64

    def validate(self) -> None:
        check(lib().octgpu_validate_lattice(self.X, self.Y, self.w))

    def sites(self) -> int:
        return self.X * self.Y

    def packed_cols(self) -> int:
        return self.X // 2

    def words_per_row(self) -> int:
        return self.X // (2 * self.w)


@dataclass(frozen=True)
class DyadicPlan:
    """rng.hpp:142-151: r = m / 2^k; ops follow the bits of m above bit 0."""

    k: int
    m: int

    @property
    def ops(self) -> list[str]:
        return ["or" if (self.m >> i) & 1 else "and" for i in range(1, self.k)]

    def words(self) -> int:
        return self.k


@dataclass(frozen=True)
class ProbSpec:
    value: float
    mode: ProbMode
    plan: DyadicPlan = field(default_factory=lambda: DyadicPlan(0, 0))

    @staticmethod
    def resolve(r: float, forced: ProbMode | int | None = None) -> "ProbSpec":
        out = OctProb()
        check(lib().octgpu_resolve(float(r), -1 if forced is None else int(forced), C.byref(out)))
        return ProbSpec._from_c(out)

    @staticmethod
    def _from_c(c: OctProb) -> "ProbSpec":
        return ProbSpec(c.value, ProbMode(c.mode), DyadicPlan(c.k, c.m))

    def to_c(self) -> OctProb:
        return OctProb(self.value, int(self.mode), self.plan.k, self.plan.m)

    def draws_per_word(self, w: int = 64) -> int:
        c = self.to_c()
        return int(lib().octgpu_draws_per_word(C.byref(c), w))


@dataclass(frozen=True)
class UpdateParams:
    p: ProbSpec
    q: ProbSpec

    @staticmethod
    def make(p: float, q: float, pmode: ProbMode | None = None, qmode: ProbMode | None = None) -> "UpdateParams":
        return UpdateParams(ProbSpec.resolve(p, pmode), ProbSpec.resolve(q, qmode))

    def to_c(self) -> OctParams:
        return OctParams(self.p.to_c(), self.q.to_c())

    def draws_per_word(self, w: int = 64) -> int:
        """xi draws consumed per word (ξp, then ξq unless q is Zero; engine_vec.hpp:105,124-125)."""
        return self.p.draws_per_word(w) + (self.q.draws_per_word(w) if self.q.mode != ProbMode.Zero else 0)


def log_schedule(t_max: int, points_per_decade: int) -> list[int]:
    """measure.cpp:143-165, computed in liboctgpu."""
    from ._lib import ConfigError

    buf = (C.c_uint64 * 4096)()
    n = lib().octgpu_log_schedule(int(t_max), int(points_per_decade), buf, len(buf))
    if n == 0:
        raise ConfigError(lib().octgpu_last_error().decode())
    return [int(buf[i]) for i in range(min(n, len(buf)))]
