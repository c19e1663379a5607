set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "measure or heights or invariant or golden or flat or chunks" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_stripes_gpu.py -x -q -k "curl or mixed" 2>&1 | tail -2
timeout 300 python tools/measure_timer.py
