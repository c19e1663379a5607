set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "plan or graph or deep" 2>&1 | tail -25
timeout 900 python -m pytest tests/test_scale_gpu.py -x -q 2>&1 | tail -25
