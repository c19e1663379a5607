"""Where the e2e time goes (engine creation from pinned host planes, steps, D2H) at 2^16^2."""
import time
import sys
import os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00310_b200 as octgpu

X = Y = 1 << 16
lat = octgpu.LatticeConfig(X, Y)
flat = octgpu.new_flat(lat).planes
hp = torch.from_numpy(flat.view(np.int64)).pin_memory().numpy().view(np.uint64)
hs = torch.from_numpy(octgpu.RngStreamSet.derive(1, Y).states.view(np.int64)).pin_memory().numpy().view(np.uint64)
pp = torch.empty(hp.shape, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
ps = torch.empty(hs.shape, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
prm = octgpu.UpdateParams.make(1.0, 0.0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = octgpu.GpuEngine(octgpu.SlopeField(lat, hp), octgpu.RngStreamSet(1, hs))
    eng.sync()
    t1 = time.perf_counter()
    eng.step(prm, int(os.environ.get('MCS', 100)))
    eng.sync()
    t2 = time.perf_counter()
    eng.measure()
    t3 = time.perf_counter()
    eng.planes(out=pp)
    t35 = time.perf_counter()
    eng.streams(out=ps)
    t4 = time.perf_counter()
    print(f"planes {t35 - t3:.4f}  streams {t4 - t35:.4f}")
    del eng
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"create {t1-t0:.3f}  100 MCS {t2-t1:.3f}  measure {t3-t2:.4f}  d2h {t4-t3:.3f}  destroy {t5-t4:.3f}")

# raw copy rates of the same pinned buffers, for comparison
d = torch.empty(hp.shape, dtype=torch.int64, device="cuda")
src = torch.from_numpy(hp.view(np.int64))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    torch.from_numpy(pp.view(np.int64)).copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"raw H2D {hp.nbytes / (t1 - t0) / 1e9:.1f} GB/s  D2H {hp.nbytes / (t2 - t1) / 1e9:.1f} GB/s")
