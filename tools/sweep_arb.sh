# c4 (arbitrary p) under bulk register budgets: OCTGPU_ARB_MINB variants (tools/build_variant.sh)
for v in base arb5 arb6; do
  if [ $v = base ]; then L=""; else L="OCTGPU_LIB=tools/variants/$v/liboctgpu.so"; fi
  env $L timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --from-flat --no-e2e --no-cpu-baseline > gpurun_out/arb_$v.json 2>gpurun_out/arb_$v.err
  python -c "import json;d=json.load(open('gpurun_out/arb_$v.json'));print('$v', round(d['roofline']['kernel_ms'],4), round(d['value']), d.get('final_checksum'))"
done
