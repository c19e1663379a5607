"""OCTSCA01 / OCTRNG01 snapshots, byte-compatible with the reference
(snapshot.hpp:16-94, snapshot.cpp:23-70).

Layout, little-endian: "OCTSCA01", u32 X, u32 Y, u32 w, u64 t_mcs, u8 phase,
u8 bit convention (1 = bit 1 is slope +1), the 4 planes (x/even, x/odd,
y/even, y/odd; row-major; w-bit words), then optionally "OCTRNG01", u64 master
seed, u32 stream count, 4 x u64 xoshiro256++ state per stream.
"""
from __future__ import annotations

import struct

import numpy as np

from ._lib import ConfigError, IoError
from .engine import RngStreamSet, SlopeField, _word_dtype
from .params import LatticeConfig

MAGIC = b"OCTSCA01"
RNG_MAGIC = b"OCTRNG01"


def serialize_snapshot(f: SlopeField, streams: RngStreamSet | None = None) -> bytes:
    """serialize_snapshot (snapshot.hpp:69-94)."""
    c = f.cfg
    out = bytearray(MAGIC)
    out += struct.pack("<IIIQBB", c.X, c.Y, c.w, int(f.t_mcs), int(f.phase), 1)
    out += np.ascontiguousarray(f.planes, np.dtype(_word_dtype(c.w)).newbyteorder("<")).tobytes()
    if streams is not None:
        st = np.ascontiguousarray(streams.states, np.dtype("<u8"))
        out += RNG_MAGIC + struct.pack("<QI", int(streams.master_seed), st.shape[0]) + st.tobytes()
    return bytes(out)


def parse_snapshot(data: bytes) -> tuple[SlopeField, RngStreamSet | None]:
    """parse_snapshot (snapshot.cpp:23-70), with the reference's IoError messages."""
    pos = 0

    def take(n: int) -> bytes:
        nonlocal pos
        if len(data) - pos < n:
            raise IoError("snapshot truncated")
        b = data[pos:pos + n]
        pos += n
        return b

    if take(8) != MAGIC:
        raise IoError("not a snapshot file (bad magic)")
    X, Y, w, t, phase, conv = struct.unpack("<IIIQBB", take(22))
    cfg = LatticeConfig(X, Y, w)
    try:
        cfg.validate()
    except ConfigError as e:
        raise IoError(f"snapshot header invalid: {e}") from None
    if phase > 1:
        raise IoError("snapshot phase must be 0 or 1")
    if conv != 1:
        raise IoError(f"unsupported bit convention flag {conv}")
    n = cfg.words_per_row()
    dt = np.dtype(_word_dtype(w)).newbyteorder("<")
    planes = np.frombuffer(take(4 * Y * n * dt.itemsize), dt).reshape(4, Y, n).astype(_word_dtype(w))
    f = SlopeField(cfg, planes, t, phase)
    streams = None
    if pos < len(data):
        if take(8) != RNG_MAGIC:
            raise IoError("unrecognized trailing bytes after planes")
        seed, cnt = struct.unpack("<QI", take(12))
        st = np.frombuffer(take(32 * cnt), np.dtype("<u8")).reshape(cnt, 4).astype(np.uint64)
        streams = RngStreamSet(seed, st)
        if pos != len(data):
            raise IoError("trailing bytes after RNG state")
    return f, streams


def save_snapshot(path: str, f: SlopeField, streams: RngStreamSet | None = None) -> None:
    write_file(path, serialize_snapshot(f, streams))


def load_snapshot(path: str) -> tuple[SlopeField, RngStreamSet | None]:
    return parse_snapshot(read_file(path))


def write_file(path: str, data: bytes | str) -> None:  # snapshot.cpp:72-79
    try:
        with open(path, "wb") as fh:
            fh.write(data.encode() if isinstance(data, str) else data)
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


def read_file(path: str) -> bytes:  # snapshot.cpp:81-89
    try:
        with open(path, "rb") as fh:
            return fh.read()
    except OSError:
        raise IoError(f"cannot open: {path}") from None
