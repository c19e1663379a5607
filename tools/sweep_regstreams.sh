# k_mcs_deep live streams kept in registers (OCTGPU_DEEP_REG_STREAMS variants) at c2' (p = 1/2)
for v in base rs3 rs4; do
  if [ $v = base ]; then L=""; else L="OCTGPU_LIB=tools/variants/$v/liboctgpu.so"; fi
  env $L timeout 300 python bench.py --config c2h --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rs_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rs_$v.json'));print('$v', round(d['roofline']['kernel_ms'],4), d.get('final_checksum'))"
done
