# full GPU suite (scale tests first)
set -x
timeout 1500 python -m pytest tests/test_scale_gpu.py -x -q 2>&1 | tail -5
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_scale_gpu.py 2>&1 | tail -15
