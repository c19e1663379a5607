# W^2 row pass: ncu source page (per-SASS executed instruction counts) of the current kernel, rough field
set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2m_meas python tools/measure_timer.py > /dev/null 2>&1
ncu -i gpurun_out/r2m_meas.ncu-rep --page source --csv > gpurun_out/r2m_meas_source.csv 2>/dev/null
python tools/ncu_extract.py gpurun_out/r2m_meas.ncu-rep gpurun_out/r2m_ncu_meas.json --label "k_measure_rows final c2h t=200"
rm -f gpurun_out/*.ncu-rep
