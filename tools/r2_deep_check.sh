# Block-wide deep kernel: parity subset, timings, then the whole GPU suite.
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "deep or plan or graph or tile or golden" 2>&1 | tail -15
for cfg in "P=1.0 K=300" "P=1.0 K=300 OCTGPU_DEEP_L=4" "P=0.5 K=200" "P=0.0 Q=0.5 K=200" "P=0.5 Q=0.5 K=100" "X=131072 Y=131072 P=1.0 K=60" "X=131072 Y=131072 P=0.5 K=40"; do
  env $cfg TAG="$cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
timeout 1500 python -m pytest tests/test_scale_gpu.py -x -q 2>&1 | tail -5
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_scale_gpu.py 2>&1 | tail -15
