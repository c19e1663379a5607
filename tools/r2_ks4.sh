# words per ring stage 4 vs 2 with the split-phase live exchange
set -x
for v in base ks4 base ks4; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 Q=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
