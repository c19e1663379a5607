# k_mcs_deep block shape: 8 warps x 2 blocks/SM (base) vs 5 x 3 and 4 x 4 (fills the 148 SMs in one wave at L = 6)
set -x
for v in base w5 w4 base w5 w4; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=1.0 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
for v in base w5; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  X=131072 Y=131072 P=1.0 K=48 KWARM=3 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 Q=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
