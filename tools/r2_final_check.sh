# final check: full GPU suite, smoke, the driver's command line and its reference arm
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f_bench_k20.json 2> gpurun_out/r2f_bench_k20.err
python -c "import json; d=json.load(open('gpurun_out/r2f_bench_k20.json')); print('k20', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['clocks'], d['gpu_launches'])"
