set -x
for cfg in "P=0.5 Q=0.5 K=100" "P=0.5 Q=0.5 K=100 OCTGPU_DEEP=2" "P=0.75 Q=0.0 K=100" "P=0.75 Q=0.0 K=100 OCTGPU_DEEP=2" "P=0.5 Q=0.25 K=100" "P=0.5 Q=0.25 K=100 OCTGPU_DEEP=2"; do
  env $cfg TAG="$cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
