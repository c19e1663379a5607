set -x
OCTGPU_TRACE_CREATE=1 MCS=20 timeout 300 python tools/e2e_probe.py 2>&1 | tail -12
MCS=20 timeout 300 python tools/e2e_probe.py 2>&1 | tail -8
timeout 900 python -m pytest tests -x -q -m gpu -k "create or snapshot or session or dropin or set_state or resume or abi" 2>&1 | tail -2
