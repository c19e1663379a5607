set -x
timeout 900 python -m pytest tests/test_stripes_gpu.py tests/test_p2p_ipc_gpu.py tests/test_dropin_gpu.py -x -q 2>&1 | tail -4
timeout 900 python -m pytest tests/test_scale_gpu.py -x -q -k "stripes" 2>&1 | tail -2
timeout 600 python tools/stripe_overhead.py 2>&1 | tail -12
OCTGPU_FUSED_LINK=0 timeout 600 python tools/stripe_overhead.py 2>&1 | tail -12
