set -x
timeout 1500 python -m pytest tests/test_scale_gpu.py -x -q --durations=5 2>&1 | tail -12
