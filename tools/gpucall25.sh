timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/b25_default.json 2> gpurun_out/b25_default.err; tail -c 1500 gpurun_out/b25_default.json
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_deep -s 3 -c 1 -o gpurun_out/p25_c2 python bench.py --config c2 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p25_c2.ncu-rep gpurun_out/p25_c2.json --label "k_mcs_deep dp9 c2 r1"; ncu -i gpurun_out/p25_c2.ncu-rep --page source --csv > gpurun_out/p25_c2_source.csv 2>/dev/null
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_deep -s 3 -c 1 -o gpurun_out/p25_c5 python bench.py --config c5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p25_c5.ncu-rep gpurun_out/p25_c5.json --label "k_mcs_deep dp9 c5 r1"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_mcs_bulk -s 2 -c 1 -o gpurun_out/p25_c4 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/p25_c4.ncu-rep gpurun_out/p25_c4.json --label "k_mcs_bulk c4 funnel+carry r1"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c2_k30.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
