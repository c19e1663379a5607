# plane-major loads in the W^2 row pass, with table replication variants (pa = default 16/1/1/1)
set -x
for v in u32a pa pb pc pd u32a pa pb pc pd; do
  export OCTGPU_LIB=tools/variants/$v/liboctgpu.so
  echo "== $v"; timeout 300 python tools/measure_timer.py; X=131072 Y=131072 MCS=50 timeout 300 python tools/measure_timer.py
done
unset OCTGPU_LIB
timeout 900 python -m pytest tests -x -q -m gpu -k "measure or moment or W2 or heights or invariant or curl or stripe" 2>&1 | tail -3
OCTGPU_LIB=tools/variants/pa/liboctgpu.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_measure_rows -s 3 -c 1 -o gpurun_out/r2v_pa python tools/measure_timer.py > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2v_pa.ncu-rep gpurun_out/r2v_ncu_meas_pa.json --label "k_measure_rows pa c2h t=200"
rm -f gpurun_out/*.ncu-rep
