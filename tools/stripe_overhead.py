"""Cost of the device-side halo exchange, measured on ONE GPU: the 2^16 x 2^16 lattice as N row stripes,
each on its own CUDA stream, exchanging halos over (same-device) peer memory with no host synchronisation
between passes -- i.e. N 'virtual GPUs' sharing one B200 -- against the single periodic engine.
Prints ms per MCS; the difference is the exchange protocol's cost when the stripes share the SMs."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00310_b200 as octgpu  # noqa: E402
from paper_1606_00310_b200.stripes import PeerLocalTransport, StripeEngine, StripeGroup, stripe_bounds  # noqa: E402

X = Y = 1 << 16
K = int(os.environ.get("K", 200))
P = float(os.environ.get("P", 1.0))
cfg = octgpu.LatticeConfig(X, Y)
prm = octgpu.UpdateParams.make(P, 0.0)

eng = octgpu.GpuEngine(cfg, 1)
eng.step(prm, 4)
eng.sync()
t0 = time.perf_counter()
eng.step(prm, K)
eng.sync()
base = (time.perf_counter() - t0) * 1e3 / K
print(f"periodic engine: {base:.4f} ms/MCS")
del eng
for n in (2, 4, 8):
    engines, streams = [], []
    for r in range(n):
        y0, y1 = stripe_bounds(Y, n, r)
        e = StripeEngine(cfg, y0, y1, 1)
        streams.append(torch.cuda.Stream())
        e.set_stream(streams[-1].cuda_stream)
        engines.append(e)
    grp = StripeGroup(PeerLocalTransport(engines), X, Y)
    grp.step(prm, 4)
    for e in engines:
        e.sync()
    t0 = time.perf_counter()
    grp.step(prm, K)
    for e in engines:
        e.sync()
    ms = (time.perf_counter() - t0) * 1e3 / K
    print(f"{n} stripes on {n} streams (peer exchange): {ms:.4f} ms/MCS ({100 * (ms / base - 1):+.1f}% vs periodic)")
    del grp, engines
