timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/b21_default.json 2> gpurun_out/b21_default.err; tail -c 3000 gpurun_out/b21_default.json
for c in c2h c3 c4 c5; do timeout 300 python bench.py --config $c --steps 1000 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b21_$c.json; python -c "import json; d=json.load(open('gpurun_out/b21_$c.json')); print('$c', round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), round(d['ms_per_step'],4))"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c2_k30.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for c in c2 c5; do timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_deep -s 3 -c 1 -o gpurun_out/p21_$c python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p21_$c.ncu-rep gpurun_out/p21_$c.json --label "k_mcs_deep S3 $c r1"; done
ncu -i gpurun_out/p21_c2.ncu-rep --page source --csv > gpurun_out/p21_c2_source.csv 2>/dev/null
timeout 300 ncu --set full --clock-control none -k regex:k_measure_rows -c 1 -o gpurun_out/p21_meas python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p21_meas.ncu-rep gpurun_out/p21_meas.json --label "k_measure_rows c2 r1"
rm -f gpurun_out/*.ncu-rep
