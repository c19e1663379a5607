"""The W^2 row pass's 32-site unit algebra (csrc/measure.cu, tab32_entry / unit32 / flush_chunk32), restated in
Python: four chained 8-site tables whose packed 64-bit entries are summed without carries between fields, 32-bit
chunk accumulators relative to the chunk start, and the chunk decode C_k = sum over the chunk's sites of u^k
(slope_field.hpp:206-229 integration of sigma_x-, measure.cpp:24-56 power sums). CPU check of the packing ranges
and of the decode on random, all-up, all-down and biased rows; the CUDA kernel itself is pinned by the -m gpu
parity tests against the reference's reconstruction."""
import random

import pytest

BASE = [0, 0, 9, 26]  # row base of T1..T3 in the shared table (tab_base)


def tab_q(b, o):
    p = pc = 0
    q = [0, 0, 0, 0]
    for i in range(8):
        bit = (b >> (4 + (i >> 1))) & 1 if i & 1 else (b >> (i >> 1)) & 1
        p += 1 if bit else -1
        pc += bit
        v = o + p
        for k in range(4):
            q[k] += v ** (k + 1)
    return q, pc


def bias(j):
    q, _ = tab_q(0, -8 * j)  # the all-down byte at the lowest offset of table j
    return -q[0] // 2, -((q[2] - q[0]) // 6)


B1 = sum(bias(j)[0] for j in range(4))
B3 = sum(bias(j)[1] for j in range(4))


def entry(b, o, j):
    q, pc = tab_q(b, o)
    assert (q[2] - q[0]) % 6 == 0 and q[1] % 4 == 0 and q[0] % 2 == 0 and (q[3] - 4) % 16 == 0
    b1, b3 = bias(j)
    return ((q[2] - q[0]) // 6 + b3) | (q[1] // 4) << 17 | (q[0] // 2 + b1) << 29 | ((q[3] - 4) // 16) << 39 | pc << 58


T0 = [entry(b, 0, 0) for b in range(256)]
TJ = [0] * (51 * 256)
for _j in (1, 2, 3):
    for _f in range(8 * _j + 1):
        for _b in range(256):
            TJ[(BASE[_j] + _f) * 256 + _b] = entry(_b, 2 * (_f - 4 * _j), _j)


def to_bytes(bits):  # 8 sites per byte: even sites -> low nibble, odd sites -> high nibble
    out = []
    for c in range(len(bits) // 8):
        b = 0
        for i, s in enumerate(bits[8 * c:8 * c + 8]):
            if s:
                b |= (1 << (i >> 1)) if i % 2 == 0 else (1 << (4 + (i >> 1)))
        out.append(b)
    return out


def chunk_sums(bits):
    """flush_chunk32's C_1..C_4 for one chunk (<= 16 units of 32 sites), with the kernel's 32-bit range checks."""
    bys = to_bytes(bits)
    A = dict.fromkeys(["s", "s2", "s3", "s4", "f1", "f2", "f3", "f4", "sf1", "sf2", "sf3", "s2f1", "s2f2", "s3f1"], 0)
    s = 0
    widths = {"F3": 17, "F2": 12, "F1": 10, "F4": 19, "FD": 6}
    for u in range(len(bys) // 4):
        e = T0[bys[4 * u]]
        for j in (1, 2, 3):
            e += TJ[(BASE[j] + (e >> 58)) * 256 + bys[4 * u + j]]
        assert e < 1 << 64
        F = {"F3": e & 0x1ffff, "F2": (e >> 17) & 0xfff, "F1": (e >> 29) & 0x3ff, "F4": (e >> 39) & 0x7ffff,
             "FD": e >> 58}
        for k, w in widths.items():
            assert F[k] < 1 << w
        s2, s3 = s * s, s * s * s
        A["s"] += s
        A["s2"] += s2
        A["s3"] += s3
        A["s4"] += s2 * s2
        A["f1"] += F["F1"]
        A["f2"] += F["F2"]
        A["f3"] += F["F3"]
        A["f4"] += F["F4"]
        A["sf1"] += s * F["F1"]
        A["sf2"] += s * F["F2"]
        A["sf3"] += s * F["F3"]
        A["s2f1"] += s2 * F["F1"]
        A["s2f2"] += s2 * F["F2"]
        A["s3f1"] += s3 * F["F1"]
        for k in ("s", "s2", "s3", "f1", "f2", "f3", "f4", "sf1", "sf2", "sf3", "s2f1", "s2f2"):
            assert -(1 << 31) <= A[k] < 1 << 31, k  # the kernel's 32-bit accumulators
        s += F["FD"] - 16
    K = len(bys) // 4
    C1 = 64 * A["s"] + 2 * A["f1"] - 2 * B1 * K
    C2 = 128 * A["s2"] + 8 * A["sf1"] - 8 * B1 * A["s"] + 4 * A["f2"]
    C3 = (256 * A["s3"] + 24 * A["s2f1"] - 24 * B1 * A["s2"] + 24 * A["sf2"] + 6 * A["f3"] - 6 * B3 * K
          + 2 * A["f1"] - 2 * B1 * K)
    C4 = (512 * A["s4"] + 64 * A["s3f1"] - 64 * B1 * A["s3"] + 96 * A["s2f2"] + 48 * A["sf3"] - 48 * B3 * A["s"]
          + 16 * A["sf1"] - 16 * B1 * A["s"] + 16 * A["f4"] + 16 * K)
    return [C1, C2, C3, C4], 2 * s


def direct(bits):
    h, S = 0, [0, 0, 0, 0]
    for b in bits:
        h += 1 if b else -1
        for k in range(4):
            S[k] += h ** (k + 1)
    return S, h


def test_unit_biases():
    assert (B1, B3) == (264, 46376)  # kU32B1 / kU32B3 (static_assert in measure.cu)


@pytest.mark.parametrize("kind", ["random", "up", "down", "biased", "alternating", "short"])
def test_chunk_decode_matches_direct_power_sums(kind):
    rng = random.Random(7)
    for _ in range(40 if kind in ("random", "biased") else 1):
        n = 512 if kind != "short" else 32 * rng.randint(1, 15)
        if kind == "random":
            bits = [rng.randint(0, 1) for _ in range(n)]
        elif kind == "up":
            bits = [1] * n
        elif kind == "down":
            bits = [0] * n
        elif kind == "alternating":
            bits = [i & 1 for i in range(n)]
        elif kind == "short":
            bits = [rng.randint(0, 1) for _ in range(n)]
        else:
            pr = rng.random()
            bits = [1 if rng.random() < pr else 0 for _ in range(n)]
        sums, end = chunk_sums(bits)
        ref, h = direct(bits)
        assert sums == ref and end == h
