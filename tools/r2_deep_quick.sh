# quick: deep parity subset + timings
set -x
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "deep or plan" 2>&1 | tail -5
for cfg in "P=1.0 K=300" "P=1.0 K=300 OCTGPU_DEEP_L=4" "P=0.5 K=200" "P=0.0 Q=0.5 K=200" "X=131072 Y=131072 P=1.0 K=60" "X=131072 Y=131072 P=0.5 K=40"; do
  env $cfg TAG="$cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
