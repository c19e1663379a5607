set -x
for c in "c2 1.0"; do set -- $c
  P=$2 K=9 KWARM=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mcs_deep -s 2 -c 1 -o gpurun_out/r2w_$1 python tools/step_timer.py > /dev/null 2>&1
  python tools/ncu_extract.py gpurun_out/r2w_$1.ncu-rep gpurun_out/r2w_ncu_deep_$1.json --label "k_mcs_deep $1 r2w"
  ncu -i gpurun_out/r2w_$1.ncu-rep --page source --csv > gpurun_out/r2w_src_$1.csv 2>/dev/null
  rm -f gpurun_out/r2w_$1.ncu-rep
done
