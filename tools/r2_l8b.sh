set -x
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_counter_gpu.py -x -q -k "deep or plan or graph or tile or counter" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_scale_gpu.py -x -q -k "c2" 2>&1 | tail -3
for cfg in "P=1.0 K=20 KWARM=9980" "P=1.0 K=20 KWARM=9980 OCTGPU_DEEP_LONG=0" "P=1.0 K=300" "X=131072 Y=131072 P=1.0 K=60"; do
  env $cfg TAG="$cfg" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-configs --no-cpu-baseline > gpurun_out/r2l8_k20.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2l8_k20.json')); print('k20', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['gpu_launches'])"
