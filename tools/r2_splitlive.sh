# split-phase exchange for the one-draw live passes only (c2'), vs HEAD
set -x
for v in base git_head base git_head; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.0 Q=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=1.0 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 Q=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
unset OCTGPU_LIB
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q -k "deep or c2h or c2rough or c2h200 or plan" 2>&1 | tail -2
