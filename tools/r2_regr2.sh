set -x
for K in 198 200 196 202 400; do
  P=0.5 K=$K TAG=base timeout 300 python tools/step_timer.py 2>&1 | tail -1
  OCTGPU_LIB=tools/variants/l6m1/liboctgpu.so P=0.5 K=$K TAG=l6m1 timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
