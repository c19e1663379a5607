# c2' regression hunt: in-tree vs fresh build vs engine.cu before the pooled small buffers
set -x
for v in base cur prevalloc base cur prevalloc; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=0.5 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=1.0 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
