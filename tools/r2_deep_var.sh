# A/B: deep kernel variants (tools/variants/*), c2 / c2h / c5 timings
set -x
for v in default $VARIANTS; do
  if [ $v = default ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  for cfg in "P=1.0 K=300" "P=0.5 K=200" "X=131072 Y=131072 P=1.0 K=60"; do
    env $cfg TAG="$v $cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
  done
done
