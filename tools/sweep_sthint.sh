# plane-store cache operator of the fused kernels (OCTGPU_ST_HINT variants): default write-back vs .cs (evict-first)
for v in base stcs base stcs; do
  if [ $v = base ]; then L=""; else L="OCTGPU_LIB=tools/variants/$v/liboctgpu.so"; fi
  for c in c2 c3; do
    env $L timeout 300 python bench.py --config $c --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sh_$v_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/sh_$v_$c.json'));print('$v $c', round(d['roofline']['kernel_ms'],4), d.get('final_checksum'))"
  done
done
