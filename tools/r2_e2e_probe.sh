set -x
OCTGPU_TRACE_CREATE=1 MCS=20 timeout 300 python tools/e2e_probe.py 2>&1 | tail -24
