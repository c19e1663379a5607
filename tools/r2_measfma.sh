# W^2 row pass: accumulator adds and field extractions on the FMA pipe (default) vs the ALU pipe (nofma)
set -x
for v in base nofma base nofma; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  echo "== $v"; timeout 300 python tools/measure_timer.py; X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
  P=1.0 MCS=7 timeout 300 python tools/measure_timer.py
done
unset OCTGPU_LIB
timeout 900 python -m pytest tests -x -q -m gpu -k "measure or moment or W2 or heights or invariant or curl" 2>&1 | tail -2
