# k_mcs_bulk consumer warps per block (OCTGPU_BULK_WARPS variants built by tools/build_variant.sh)
for v in base bulk5 bulk6; do
  if [ $v = base ]; then L=""; else L="OCTGPU_LIB=tools/variants/$v/liboctgpu.so"; fi
  for c in c2h c3 c4; do
    S=200; [ $c = c4 ] && S=20
    env $L OCTGPU_DEEP=0 timeout 300 python bench.py --config $c --steps $S --warmup 3 --from-flat --no-e2e --no-cpu-baseline > gpurun_out/kp_${v}_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/kp_${v}_$c.json'));print('$v $c', round(d['roofline']['kernel_ms'],4), d.get('final_checksum'))"
  done
done
