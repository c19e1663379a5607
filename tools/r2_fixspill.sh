# live 2-MCS pass after the link_signal barrier fix (spill-free again): c2', c3, c2 and the old build
set -x
for v in base git_1f4032b base; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=0.5 Q=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
  P=1.0 K=198 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
unset OCTGPU_LIB
timeout 900 python -m pytest tests -x -q -m gpu -k "stripe or p2p or link" 2>&1 | tail -2
