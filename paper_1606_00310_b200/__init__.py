"""octsca-b200: B200-native bit-vectorized SCA for the 2+1-D octahedron model.

Drop-in for the reference engine's hot path (octsca::VecEngine step loop and
W² measurement, arXiv:1606.00310). The compute runs in liboctgpu.so
(hand-written sm_100a CUDA behind the C-ABI in include/octgpu.h); this
package is the host-side mirror of the reference interface.
"""
from ._lib import ConfigError, CudaError, InvariantError, IoError, OctError
from .engine import (GpuEngine, HeightMap, MeasurementRecord, RngStreamSet, SlopeField, field_checksum,
                     new_flat, release_pool)
from .params import DyadicPlan, LatticeConfig, ProbMode, ProbSpec, UpdateParams, log_schedule
from .run import run

__all__ = [
    "ConfigError", "CudaError", "InvariantError", "IoError", "OctError", "GpuEngine", "HeightMap",
    "MeasurementRecord", "RngStreamSet", "SlopeField", "field_checksum", "new_flat", "release_pool", "DyadicPlan",
    "LatticeConfig", "ProbMode", "ProbSpec", "UpdateParams", "log_schedule", "run",
]
__version__ = "0.1.0"
