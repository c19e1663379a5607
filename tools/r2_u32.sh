# 32-site units in the W^2 row pass: A/B against 16-site units, then the measurement parity tests
set -x
for v in u16 u32 u16 u32; do
  export OCTGPU_LIB=tools/variants/$v/liboctgpu.so
  echo "== $v"; timeout 300 python tools/measure_timer.py; X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
  P=1.0 MCS=7 timeout 300 python tools/measure_timer.py
done
unset OCTGPU_LIB
timeout 900 python -m pytest tests -x -q -m gpu -k "measure or moment or W2 or heights or invariant or curl" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_scale_gpu.py -x -q 2>&1 | tail -3
