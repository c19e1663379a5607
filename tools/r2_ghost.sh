set -x
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "deep_vs_oracle or tile or graph" 2>&1 | tail -2
for g in kernel memcpy kernel memcpy; do
for cfg in "P=1.0 K=300" "P=0.5 K=200"; do
  env $cfg OCTGPU_GHOST=$g TAG="$g $cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done; done
