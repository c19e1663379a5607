# A/B: deep ring words/stage (KS) x stages (S)
set -x
for v in ks2 ks4; do
  export OCTGPU_LIB=tools/variants/$v/liboctgpu.so
  for S in 2 3 4 5; do
    for cfg in "P=1.0 K=300" "P=0.5 K=200"; do
      env $cfg OCTGPU_DEEP_S=$S TAG="$v S=$S $cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
    done
  done
done
