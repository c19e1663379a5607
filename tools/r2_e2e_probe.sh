set -x
OCTGPU_TRACE_CREATE=1 timeout 300 python tools/e2e_probe.py 2>&1 | tail -40
