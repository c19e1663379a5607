timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c2 c2h c3 c4 c5; do timeout 300 python bench.py --config $c --steps 300 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b30_$c.json; python -c "import json; d=json.load(open('gpurun_out/b30_$c.json')); print('$c', round(d['value']), round(d['roofline']['kernel_ms'],4), d['final_checksum'])"; done
