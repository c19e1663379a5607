timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in c4 c2h c3; do timeout 300 python bench.py --config $c --steps 300 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b22_$c.json; python -c "import json; d=json.load(open('gpurun_out/b22_$c.json')); print('$c', round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"; done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_bulk -s 2 -c 1 -o gpurun_out/p22_c4 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p22_c4.ncu-rep gpurun_out/p22_c4.json --label "k_mcs_bulk c4 imad-rot r1"
rm -f gpurun_out/*.ncu-rep
