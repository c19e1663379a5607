set -x
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_counter_gpu.py -x -q -k "deep or plan or graph or tile or counter" 2>&1 | tail -2
for cfg in "P=1.0 K=300" "P=0.5 K=200" "P=0.5 Q=0.5 K=100" "X=131072 Y=131072 P=1.0 K=60"; do
  env $cfg TAG="$cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
