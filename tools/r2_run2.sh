set -x
export OCTGPU_TRACE_CREATE=1
timeout 600 python tools/e2e_probe.py 2>&1 | tail -30
unset OCTGPU_TRACE_CREATE
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/measure_timer.py
MCS=2000 timeout 300 python tools/measure_timer.py
P=1.0 MCS=100 timeout 300 python tools/measure_timer.py
X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2b_meas python tools/measure_timer.py > /dev/null 2>&1; python tools/ncu_extract.py gpurun_out/r2b_meas.ncu-rep gpurun_out/r2b_ncu_k_measure_rows_c2h.json --label "k_measure_rows c2h r2b"; cat gpurun_out/r2b_ncu_k_measure_rows_c2h.json
