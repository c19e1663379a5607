set -x
OCTGPU_TRACE_CREATE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e2etrace.json 2> gpurun_out/r2e2etrace.err
grep -n "upload" -A12 gpurun_out/r2e2etrace.err | tail -40
