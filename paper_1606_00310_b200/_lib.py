"""ctypes binding of liboctgpu.so (include/octgpu.h).

The library is built in-tree (``paper_1606_00310_b200/csrc/liboctgpu.so``) by
``__graft_entry__.build()`` / ``make -C paper_1606_00310_b200/csrc``. There is
no fallback: if the library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# OCTGPU_LIB: a development build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("OCTGPU_LIB") or os.path.join(HERE, "csrc", "liboctgpu.so")


class OctError(RuntimeError):
    """Base class; subclasses mirror octsca's exceptions (errors.hpp:8-25)."""

    exit_code = 5


class ConfigError(OctError):
    exit_code = 1


class InvariantError(OctError):
    exit_code = 2


class IoError(OctError):
    exit_code = 3


class CudaError(OctError):
    exit_code = 4


_ERRORS = {1: ConfigError, 2: InvariantError, 3: IoError, 4: CudaError}


class OctProb(C.Structure):
    _fields_ = [("value", C.c_double), ("mode", C.c_int32), ("k", C.c_uint32), ("m", C.c_uint64)]


class OctParams(C.Structure):
    _fields_ = [("p", OctProb), ("q", OctProb)]


class OctMoments(C.Structure):
    _fields_ = [
        ("t", C.c_uint64),
        ("n_sites", C.c_uint64),
        ("s_lo", C.c_uint64 * 4),
        ("s_hi", C.c_int64 * 4),
        ("W2", C.c_double),
        ("mean_h", C.c_double),
        ("skew", C.c_double),
        ("kurt", C.c_double),
    ]


class OctStripeMoments(C.Structure):
    _fields_ = [
        ("t", C.c_uint64),
        ("n_sites", C.c_uint64),
        ("s_lo", C.c_uint64 * 4),
        ("s_hi", C.c_int64 * 4),
        ("col_sum", C.c_int64),
        ("sy_first", C.c_int64),
        ("row_first_sum", C.c_int64),
        ("curl_count", C.c_uint64),
        ("curl_first", C.c_uint64),
    ]


class OctPeer(C.Structure):
    _fields_ = [
        ("planes", C.c_uint64 * 2),
        ("rng", C.c_uint64 * 2),
        ("done", C.c_uint64),
        ("alloc_rows", C.c_uint32),
        ("rows", C.c_uint32),
        ("n", C.c_uint32),
        ("w", C.c_uint32),
        ("device", C.c_int32),
        ("pad", C.c_int32),
    ]


IPC_BYTES = 512  # OCTGPU_IPC_BYTES

# Every symbol include/octgpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "octgpu_resolve", "octgpu_draws_per_word", "octgpu_validate_lattice", "octgpu_stream_states",
    "octgpu_log_schedule", "octgpu_create", "octgpu_create_from", "octgpu_set_state", "octgpu_destroy", "octgpu_set_stream",
    "octgpu_sync", "octgpu_step", "octgpu_sweep", "octgpu_t", "octgpu_phase", "octgpu_master_seed",
    "octgpu_get_planes", "octgpu_get_states", "octgpu_field_checksum", "octgpu_measure", "octgpu_heights",
    "octgpu_last_error", "octgpu_version", "octgpu_launch_count", "octgpu_create_stripe", "octgpu_stripe_sizes",
    "octgpu_halo_pack", "octgpu_halo_unpack", "octgpu_stripe_mcs", "octgpu_stripe_mcs_n", "octgpu_stripe_max_mcs",
    "octgpu_stripe_finish", "octgpu_measure_stripe", "octgpu_stripe_peer", "octgpu_stripe_ipc_export",
    "octgpu_stripe_ipc_open", "octgpu_stripe_connect", "octgpu_stripe_pass", "octgpu_stripe_pull",
    "octgpu_stripe_disconnect", "octgpu_set_tile_shift", "octgpu_stripes_combine",
    "octgpu_set_rng", "octgpu_get_rng",
    "octgpu_stripe_y0", "octgpu_stripe_rows", "octgpu_height_moments", "octgpu_release_pool",
    "octgpu_balances", "octgpu_pass_plan",
)

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                          f"(make -C paper_1606_00310_b200/csrc). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    P = C.POINTER
    sig = {
        "octgpu_resolve": (i32, [dbl, i32, P(OctProb)]),
        "octgpu_draws_per_word": (u32, [P(OctProb), u32]),
        "octgpu_validate_lattice": (i32, [u32, u32, u32]),
        "octgpu_stream_states": (i32, [u64, u32, vp]),
        "octgpu_log_schedule": (u32, [u64, u32, vp, u32]),
        "octgpu_create": (i32, [u32, u32, u32, u64, i32, P(vp)]),
        "octgpu_create_from": (i32, [u32, u32, u32, u64, i32, vp, vp, u32, u64, i32, P(vp)]),
        "octgpu_set_state": (i32, [vp, u64, i32, vp, vp, u32]),
        "octgpu_destroy": (None, [vp]),
        "octgpu_set_stream": (i32, [vp, vp]),
        "octgpu_sync": (i32, [vp]),
        "octgpu_step": (i32, [vp, P(OctParams), u64]),
        "octgpu_sweep": (i32, [vp, i32, P(OctParams), vp]),
        "octgpu_t": (u64, [vp]),
        "octgpu_phase": (i32, [vp]),
        "octgpu_master_seed": (u64, [vp]),
        "octgpu_get_planes": (i32, [vp, vp]),
        "octgpu_get_states": (i32, [vp, vp]),
        "octgpu_field_checksum": (i32, [vp, P(u64)]),
        "octgpu_measure": (i32, [vp, P(OctMoments)]),
        "octgpu_heights": (i32, [vp, vp]),
        "octgpu_last_error": (C.c_char_p, []),
        "octgpu_version": (C.c_char_p, []),
        "octgpu_launch_count": (u64, [vp]),
        "octgpu_create_stripe": (i32, [u32, u32, u32, u32, u32, u64, i32, vp, vp, u64, i32, P(vp)]),
        "octgpu_stripe_sizes": (i32, [vp, P(u64), P(u64), P(u64)]),
        "octgpu_halo_pack": (i32, [vp, vp, vp]),
        "octgpu_halo_unpack": (i32, [vp, vp, vp]),
        "octgpu_stripe_mcs": (i32, [vp, P(OctParams), vp]),
        "octgpu_stripe_mcs_n": (i32, [vp, P(OctParams), u32, vp]),
        "octgpu_stripe_max_mcs": (i32, [vp, P(OctParams)]),
        "octgpu_stripe_peer": (i32, [vp, P(OctPeer)]),
        "octgpu_stripe_ipc_export": (i32, [vp, vp]),
        "octgpu_stripe_ipc_open": (i32, [vp, vp, P(OctPeer)]),
        "octgpu_stripe_connect": (i32, [vp, P(OctPeer), P(OctPeer)]),
        "octgpu_stripe_pass": (i32, [vp, P(OctParams), u32]),
        "octgpu_stripe_pull": (i32, [vp]),
        "octgpu_stripe_disconnect": (i32, [vp]),
        "octgpu_set_tile_shift": (i32, [vp, u64]),
        "octgpu_set_rng": (i32, [vp, i32]),
        "octgpu_get_rng": (i32, [vp]),
        "octgpu_stripes_combine": (i32, [P(OctStripeMoments), u32, u32, u32, P(OctMoments)]),
        "octgpu_stripe_finish": (i32, [vp, vp]),
        "octgpu_measure_stripe": (i32, [vp, P(OctStripeMoments)]),
        "octgpu_stripe_y0": (u32, [vp]),
        "octgpu_stripe_rows": (u32, [vp]),
        "octgpu_height_moments": (None, [u32, u32, vp, vp]),
        "octgpu_release_pool": (i32, [i32]),
        "octgpu_balances": (i32, [vp, vp, vp]),
        "octgpu_pass_plan": (i32, [vp, P(OctParams), P(i32), P(i32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc:
        msg = lib().octgpu_last_error().decode()
        raise _ERRORS.get(rc, OctError)(msg)
