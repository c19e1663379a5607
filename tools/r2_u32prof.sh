# ncu of k_measure_rows, 16- vs 32-site units (rough field p = 1/2 t = 200)
set -x
for v in u16 u32; do
  OCTGPU_LIB=tools/variants/$v/liboctgpu.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2v_$v python tools/measure_timer.py > /dev/null 2>&1
  python tools/ncu_extract.py gpurun_out/r2v_$v.ncu-rep gpurun_out/r2v_ncu_meas_$v.json --label "k_measure_rows $v c2h t=200"
  ncu -i gpurun_out/r2v_$v.ncu-rep --page source --csv > gpurun_out/r2v_src_$v.csv 2>/dev/null
  ncu -i gpurun_out/r2v_$v.ncu-rep --page raw --csv > gpurun_out/r2v_raw_$v.csv 2>/dev/null
  rm -f gpurun_out/r2v_$v.ncu-rep
done
