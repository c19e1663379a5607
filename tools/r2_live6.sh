# 3-MCS passes (L = 6) for one-draw live streams (p = 1/2): parked / register / one-block-per-SM variants
set -x
for v in base l6r4 l6r6 l6m1 base l6r4 l6r6 l6m1; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=0.5 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
