# Round evidence: GPU tests, smoke, the default bench line, per-config lines, ncu captures, launch list.
#   gpurun --timeout 2400 -- 'bash tools/gpu_evidence.sh TAG'
TAG=${1:-r1}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; tail -c 400 gpurun_out/${TAG}_bench_default.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_reference.json
for c in c2h c3 c4 c5; do timeout 300 python bench.py --config $c --steps 1000 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$c.json; python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_$c.json')); print('$c', round(d['value']), round(d['roofline']['kernel_ms'],4))"; done
timeout 300 python bench.py --config c3 --rng counter --steps 1000 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c3_counter.json; python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_c3_counter.json')); print('c3 counter', round(d['value']), round(d['roofline']['kernel_ms'],4))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c2_k30.csv python bench.py --steps 30 --warmup 3 --from-flat --no-cpu-baseline --no-e2e > /dev/null 2>&1
for c in c2 c2h c3 c5; do timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_deep -s 3 -c 1 -o gpurun_out/${TAG}_deep_$c python bench.py --config $c --steps 40 --warmup 3 --from-flat --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/${TAG}_deep_$c.ncu-rep gpurun_out/${TAG}_ncu_k_mcs_deep_$c.json --label "k_mcs_deep $c $TAG"; done
for c in c4; do timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_bulk -s 2 -c 1 -o gpurun_out/${TAG}_bulk_$c python bench.py --config $c --steps 4 --warmup 3 --from-flat --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/${TAG}_bulk_$c.ncu-rep gpurun_out/${TAG}_ncu_k_mcs_bulk_$c.json --label "k_mcs_bulk $c $TAG"; done
timeout 300 ncu --set full --clock-control none -k regex:k_measure_rows -c 1 -o gpurun_out/${TAG}_meas python bench.py --config c2 --steps 2 --warmup 3 --from-flat --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/${TAG}_meas.ncu-rep gpurun_out/${TAG}_ncu_k_measure_rows_c2.json --label "k_measure_rows c2 $TAG"
ncu -i gpurun_out/${TAG}_deep_c2.ncu-rep --page source --csv > gpurun_out/${TAG}_deep_c2_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
# the driver's own command line (K = 20, W = 5) and its reference arm
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_k20.json 2> gpurun_out/${TAG}_bench_k20.err; python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_k20.json')); print('k20', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']))"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_reference_k20.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_reference_k20.json
