# 32-site units: table replication A/B (u32a: T0 x16 only, u32b: 8/4/2/1 (default), u32c: 16/4/1/1; u16 = 16-site units)
set -x
for v in u16 u32a u32b u32c u32a u32b u32c; do
  export OCTGPU_LIB=tools/variants/$v/liboctgpu.so
  echo "== $v"; timeout 300 python tools/measure_timer.py; X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
done
unset OCTGPU_LIB
timeout 900 python -m pytest tests -x -q -m gpu -k "measure or moment or W2 or heights or invariant or curl" 2>&1 | tail -3
OCTGPU_LIB=tools/variants/u32b/liboctgpu.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2v_u32b python tools/measure_timer.py > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2v_u32b.ncu-rep gpurun_out/r2v_ncu_meas_u32b.json --label "k_measure_rows u32b c2h t=200"
ncu -i gpurun_out/r2v_u32b.ncu-rep --page source --csv > gpurun_out/r2v_src_u32b.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
