timeout 600 python -m pytest tests/test_stripes_gpu.py -m gpu -q -x 2>&1 | tail -5
timeout 600 python -m pytest tests/test_p2p_ipc_gpu.py -m gpu -q -x 2>&1 | tail -15
