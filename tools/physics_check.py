"""KPZ / EW growth on the GPU engine (SPEC.md acceptance 3 and 4): prints beta and r^2."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_acceptance_gpu import _linfit, _mean_w2  # noqa: E402

L = int(os.environ.get("L", 1024)); seeds = int(os.environ.get("SEEDS", 10)); tmax = int(os.environ.get("TMAX", 2000))
rows = []
for rng in os.environ.get("RNG", "xoshiro,counter").split(","):
    for p, q in [(0.5, 0.0), (0.5, 0.5)]:
        t, w2 = _mean_w2(L, p, q, range(1, seeds + 1), tmax, rng=rng)
        sel = (t >= 50) & (t <= 2000)
        beta, _, rb = _linfit(np.log(t[sel]), 0.5 * np.log(w2[sel]))
        _, _, r2 = _linfit(np.log(t[sel]), w2[sel])
        print(f"{rng} L={L} p={p} q={q} seeds={seeds}: beta={beta:.4f} (loglog r2 {rb:.4f}), "
              f"W2-vs-ln t r2={r2:.4f}, W2(tmax)={w2[-1]:.3f}")
        rows.append({"rng": rng, "L": L, "p": p, "q": q, "seeds": seeds, "beta": beta, "loglog_r2": rb,
                     "w2_vs_lnt_r2": r2, "W2_tmax": float(w2[-1])})
if os.environ.get("OUT"):
    import json
    json.dump({"note": "SPEC acceptance 3 (KPZ beta = 0.24 +- 0.03 on t in [50, 2000]) and 4 (EW: W2 linear in "
                       "ln t), mean W2 over seeds, tools/physics_check.py", "rows": rows},
              open(os.environ["OUT"], "w"), indent=1)
