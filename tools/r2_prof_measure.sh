# ncu of the W^2 row kernel at 2^16^2 (p = 1/2, t = 200)
set -x
timeout 300 python tools/measure_timer.py
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2d_meas python tools/measure_timer.py > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2d_meas.ncu-rep gpurun_out/r2d_ncu_k_measure_rows.json --label "k_measure_rows c2h t=200 r2d"
ncu -i gpurun_out/r2d_meas.ncu-rep --page source --csv > gpurun_out/r2d_meas_source.csv 2>/dev/null
ncu -i gpurun_out/r2d_meas.ncu-rep --page details --csv > gpurun_out/r2d_meas_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
