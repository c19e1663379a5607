# new k_measure_rows: parity (measurement tests) + timing + ncu
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "heights" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_scale_gpu.py -x -q -k "c2h or c3" 2>&1 | tail -2
timeout 300 python tools/measure_timer.py
X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2u_meas python tools/measure_timer.py > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2u_meas.ncu-rep gpurun_out/r2u_ncu_k_measure_rows.json --label "k_measure_rows v3f c2h t=200"
ncu -i gpurun_out/r2u_meas.ncu-rep --page source --csv > gpurun_out/r2u_meas_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
