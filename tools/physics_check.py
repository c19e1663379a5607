"""KPZ / EW growth on the GPU engine (SPEC.md acceptance 3 and 4): prints beta and r^2."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_acceptance_gpu import _linfit, _mean_w2  # noqa: E402

L = int(os.environ.get("L", 1024)); seeds = int(os.environ.get("SEEDS", 10)); tmax = int(os.environ.get("TMAX", 2000))
for p, q in [(0.5, 0.0), (0.5, 0.5)]:
    t, w2 = _mean_w2(L, p, q, range(1, seeds + 1), tmax)
    sel = (t >= 50) & (t <= 2000)
    beta, _, rb = _linfit(np.log(t[sel]), 0.5 * np.log(w2[sel]))
    _, _, r2 = _linfit(np.log(t[sel]), w2[sel])
    print(f"L={L} p={p} q={q} seeds={seeds}: beta={beta:.4f} (loglog r2 {rb:.4f}), W2-vs-ln t r2={r2:.4f}, W2(tmax)={w2[-1]:.3f}")
