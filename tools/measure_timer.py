"""CUDA-event time of one W^2 measurement (octgpu_measure: rows kernel + final reduction + result D2H) at
2^16 x 2^16 (X, Y, P, Q, MCS env), after MCS steps from the flat start; also prints the exact sums."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00310_b200 as octgpu  # noqa: E402

X = int(os.environ.get("X", 1 << 16))
Y = int(os.environ.get("Y", 1 << 16))
P, Q = float(os.environ.get("P", 0.5)), float(os.environ.get("Q", 0.0))
MCS = int(os.environ.get("MCS", 200))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), 1)
eng.set_stream(stream.cuda_stream)
eng.step(octgpu.UpdateParams.make(P, Q), MCS)
eng.sync()
for _ in range(3):
    eng.measure()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    rec = eng.measure()
    b.record(stream)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"measure {X}x{Y} p={P} q={Q} t={eng.t}: median {ts[len(ts) // 2]:.4f} ms, min {ts[0]:.4f} ms; "
      f"W2={rec.W2:.12g} sums={rec.power_sums}")
