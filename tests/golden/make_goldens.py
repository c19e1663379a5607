"""Regenerate tests/golden/goldens.json from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libocref.so, built from
/root/reference/proj by oracle/Makefile). The JSON it writes is committed so
that the CPU and GPU test suites never need /root/reference at run time.

    python tests/golden/make_goldens.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Oracle, RefEngine, RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "goldens.json")

# (X, Y, w, p, q, seed, mcs)
RUNS = [
    # SURVEY.md Appendix A (1024^2, 1000 MCS) — BASELINE configs[0] and variants
    (1024, 1024, 64, 1.0, 0.0, 1, 1000),
    (1024, 1024, 64, 1.0, 0.0, 42, 1000),
    (1024, 1024, 64, 0.5, 0.0, 1, 1000),
    (1024, 1024, 64, 0.5, 0.0, 42, 1000),
    (1024, 1024, 64, 0.5, 0.5, 1, 1000),
    (1024, 1024, 64, 0.5, 0.5, 42, 1000),
    (1024, 1024, 64, 0.98, 0.02, 1, 1000),
    (1024, 1024, 64, 0.98, 0.02, 42, 1000),
    (1024, 1024, 64, 0.75, 0.0, 1, 1000),
    # SPEC.md acceptance #1 geometry (256^2, 200 MCS)
    (256, 256, 64, 0.5, 0.0, 12345, 200),
    (256, 256, 64, 0.75, 0.0, 12345, 200),
    (256, 256, 64, 0.95, 0.0, 12345, 200),
    (256, 256, 64, 0.5, 0.5, 12345, 200),
    (256, 256, 64, 0.98, 0.02, 12345, 200),
    # edge geometries: single-word rows (PBC seam inside one word), odd word
    # count, partial warps, Y = 2
    (128, 2, 64, 0.5, 0.0, 3, 50),
    (128, 30, 64, 0.5, 0.25, 3, 50),
    (128, 34, 64, 0.8125, 0.0, 3, 50),
    (384, 62, 64, 0.5, 0.5, 5, 40),
    (256, 94, 64, 0.98, 0.02, 5, 10),
    (640, 66, 64, 1.0, 0.5, 9, 20),
    (256, 64, 64, 0.0, 0.5, 9, 40),
    (256, 64, 64, 1.0, 1.0, 9, 5),
    # w = 32 (optional reference word size)
    (128, 64, 32, 0.5, 0.0, 1, 60),
    (192, 32, 32, 0.75, 0.25, 2, 30),
    (64, 34, 32, 0.95, 0.0, 4, 10),
]

SESSIONS = [  # run_session(X=Y=1024, w=64, seed=1, t_max=1000, ppd=8)
    (1024, 1024, 64, 0.5, 0.0, 1, 1000, 8),
    (1024, 1024, 64, 1.0, 0.0, 1, 1000, 8),
    (256, 256, 64, 0.5, 0.5, 7, 300, 5),
]


def main() -> None:
    o, r = Oracle(), RefLib()
    g: dict = {"source": "unmodified reference /root/reference/proj via oracle/_ref/libocref.so"}

    st = np.zeros(4, np.uint64)
    r.L.ocref_rng_from_seed(1, st)
    nxt = np.zeros(4, np.uint64)
    s2 = st.copy()
    r.L.ocref_rng_next(s2, nxt, 4)
    ss = np.zeros((3, 4), np.uint64)
    r.L.ocref_stream_set(1, 3, ss)
    j = st.copy()
    r.L.ocref_rng_jump(j)
    g["kat"] = {
        "from_seed_1": [hex(int(v)) for v in st],
        "next4": [hex(int(v)) for v in nxt],
        "stream_set_1_3": [[hex(int(v)) for v in row] for row in ss],
        "jump_from_seed_1": [hex(int(v)) for v in j],
    }
    xi = []
    for (rv, forced, w) in [(0.5, -1, 64), (0.75, -1, 64), (0.8125, -1, 64), (0.95, -1, 64), (0.02, -1, 64),
                            (1.0, -1, 64), (0.5, 3, 64), (0.5, -1, 32), (0.375, -1, 32), (0.98, -1, 32)]:
        s = np.zeros(4, np.uint64)
        r.L.ocref_rng_from_seed(7, s)
        out = np.zeros(8, np.uint64)
        r.check(r.L.ocref_xi_words(s, rv, forced, w, out, 8))
        xi.append({"r": rv, "forced": forced, "w": w, "seed": 7, "words": [hex(int(v)) for v in out],
                   "state_after": [hex(int(v)) for v in s]})
    g["xi_words"] = xi

    import ctypes as C
    res = []
    for (rv, forced) in [(0.0, -1), (0.5, -1), (0.75, -1), (0.8125, -1), (0.25, -1), (0.375, -1), (0.95, -1),
                         (1.0, -1), (0.02, -1), (2 ** -16, -1), (2 ** -17, -1), (0.5, 2), (0.5, 3), (0.75, 3),
                         (0.3, 2), (0.3, 1), (0.0, 3), (1.5, -1), (-0.1, -1), (0.0, 0), (0.5, 0), (0.2, 0)]:
        mode, dr, k, m = C.c_int(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        rc = r.L.ocref_resolve(rv, forced, 64, C.byref(mode), C.byref(dr), C.byref(k), C.byref(m))
        res.append({"r": rv, "forced": forced, "rc": rc, "mode": mode.value if rc == 0 else None,
                    "draws": dr.value if rc == 0 else None, "k": k.value if rc == 0 else None,
                    "m": m.value if rc == 0 else None, "err": r.err() if rc else None})
    g["resolve"] = res

    g["log_schedule"] = {f"{t},{p}": o.log_schedule(t, p) for (t, p) in [(10000, 8), (1000, 8), (1, 1), (7, 3),
                                                                          (100, 1), (50, 20)]}

    runs = []
    for (X, Y, w, p, q, seed, mcs) in RUNS:
        e = RefEngine(r, X, Y, seed, w=w, workers=8)
        e.step(p, q, mcs)
        h = e.heights()
        rec = e.measure()
        S = o.power_sums(h)
        runs.append({"X": X, "Y": Y, "w": w, "p": p, "q": q, "seed": seed, "mcs": mcs,
                     "checksum": hex(e.checksum()), "states_digest": hex(o.states_digest(e.states())),
                     "W2": rec[0], "mean_h": rec[1], "skew": rec[2], "kurt": rec[3],
                     "power_sums": [str(v) for v in S]})
        print("run", X, Y, w, p, q, seed, mcs, runs[-1]["checksum"], flush=True)
    g["runs"] = runs

    sessions = []
    for (X, Y, w, p, q, seed, tmax, ppd) in SESSIONS:
        with tempfile.TemporaryDirectory() as d:
            r.check(r.L.ocref_run_session(X, Y, w, p, q, seed, 8, tmax, ppd, b"vec", d.encode(), b""))
            csv = open(os.path.join(d, "measurements.csv")).read()
            snap = open(os.path.join(d, "final.snap"), "rb").read()
        sessions.append({"X": X, "Y": Y, "w": w, "p": p, "q": q, "seed": seed, "tmax": tmax, "ppd": ppd,
                         "csv": csv, "csv_sha256": hashlib.sha256(csv.encode()).hexdigest(),
                         "snap_sha256": hashlib.sha256(snap).hexdigest(), "snap_bytes": len(snap)})
        print("session", X, p, q, sessions[-1]["csv_sha256"][:16], flush=True)
    g["sessions"] = sessions

    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
