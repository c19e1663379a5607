# split-phase edge exchange in k_mcs_deep (mbarrier publish / collect around the next word's first sweep)
set -x
for v in base git_head base git_head; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=1.0 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=1.0 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 Q=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
unset OCTGPU_LIB
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "deep" 2>&1 | tail -2
