# c2' in the bench window (last 10^3 MCS of the 10^4 job, with its W^2 points): split exchange vs the r2d build
set -x
for v in base git_r2d base git_r2d; do
  if [ $v = base ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  timeout 300 python bench.py --config c2h --steps 1000 --warmup 3 --no-cpu-baseline --no-e2e --no-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['roofline']['kernel_ms'],4), d['ms_per_step'])"
  P=0.5 K=200 KWARM=9000 TAG=$v timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
