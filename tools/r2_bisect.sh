set -x
for v in git_1f4032b git_e62fffa git_8faff15 git_2584a15 base git_1f4032b base; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  P=0.5 K=200 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
