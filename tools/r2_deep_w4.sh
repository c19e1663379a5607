set -x
OCTGPU_LIB=tools/variants/w4/liboctgpu.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "deep or plan" 2>&1 | tail -2
VARIANTS="w4" bash tools/r2_deep_var.sh
