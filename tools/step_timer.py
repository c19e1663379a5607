"""Time eng.step(prm, K) in one call (all temporally blocked passes) with CUDA events."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00310_b200 as octgpu

X = int(os.environ.get("X", 1 << 16)); Y = int(os.environ.get("Y", 1 << 16)); K = int(os.environ.get("K", 300))
p, q = float(os.environ.get("P", 1.0)), float(os.environ.get("Q", 0.0))
eng = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), 1)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
prm = octgpu.UpdateParams.make(p, q)
eng.step(prm, int(os.environ.get("KWARM", 6)))
eng.sync()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
eng.step(prm, K)
b.record(st)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / K
print(f"{os.environ.get('TAG', '')} X={X} Y={Y} p={p} q={q}: {ms:.4f} ms/MCS, {X * Y / ms / 1e6:.0f} upd/ns, checksum {eng.checksum() if X * Y <= 1 << 32 else 0:#x}")
