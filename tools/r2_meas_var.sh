# A/B of the W^2 row-pass block shape (tools/build_measure_variant.sh)
set -x
for v in s16b1 s8b2 s4b4 s16b1 s8b2 s4b4; do
  export OCTGPU_LIB=tools/variants/$v/liboctgpu.so
  echo "== $v"; timeout 300 python tools/measure_timer.py; X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
done
unset OCTGPU_LIB
