set -x
OCTGPU_TRACE_CREATE=1 timeout 300 python tools/e2e_probe.py 2>&1 | tail -25
timeout 300 python bench.py --steps 20 --warmup 3 2>/dev/null | tail -1 > gpurun_out/alloc_bench.json
cat gpurun_out/alloc_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
timeout 1200 python -m pytest tests -x -q -m gpu -k "session or measure or graph or materialize or stream or api or abi" 2>&1 | tail -3
