timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -6
timeout 300 python tools/measure_timer.py
X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2c_meas python tools/measure_timer.py > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/r2c_meas.ncu-rep gpurun_out/r2c_ncu_k_measure_rows_c2h.json --label "k_measure_rows c2h r2c"; python -c "
import json; d=json.load(open('gpurun_out/r2c_ncu_k_measure_rows_c2h.json'))['kernels'][0]; print({k: d[k] for k in ['gpu__time_duration.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread']}, d['stall_pct'])"
ncu -i gpurun_out/r2c_meas.ncu-rep --page source --csv > gpurun_out/r2c_meas_source.csv 2>/dev/null; rm -f gpurun_out/*.ncu-rep
OCTGPU_TRACE_CREATE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; tail -c 600 gpurun_out/r2c_bench.json; grep -v "^$" gpurun_out/r2c_bench.err | tail -40
