timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c2 c2h c3 c4 c5; do timeout 300 python bench.py --config $c --steps 300 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b16_$c.json; python -c "import json; d=json.load(open('gpurun_out/b16_$c.json')); print('$c', round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), round(d['ms_per_step'],4))"; done
timeout 600 python bench.py > gpurun_out/b16_default.json 2> gpurun_out/b16_default.err; tail -c 2500 gpurun_out/b16_default.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c2_k30.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for c in c2 c2h c3 c4 c5; do timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_bulk -s 4 -c 1 -o gpurun_out/p16_$c python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p16_$c.ncu-rep gpurun_out/p16_$c.json --label "k_mcs_bulk(ws ks2 S2) $c r1"; done
ncu -i gpurun_out/p16_c2.ncu-rep --page source --csv > gpurun_out/p16_c2_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
