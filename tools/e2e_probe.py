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
    eng.step(prm, 100)
    eng.sync()
    t2 = time.perf_counter()
    eng.measure()
    t3 = time.perf_counter()
    eng.planes(out=pp)
    eng.streams(out=ps)
    t4 = time.perf_counter()
    del eng
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"create {t1-t0:.3f}  100 MCS {t2-t1:.3f}  measure {t3-t2:.4f}  d2h {t4-t3:.3f}  destroy {t5-t4:.3f}")
