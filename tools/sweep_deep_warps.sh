# k_mcs_deep block shape with the one-word ring: 9 compute warps x 2 blocks/SM (96 regs, default) vs
# 6 warps x 3 blocks/SM (80 regs; tools/build_variant.sh dp6 -DOCTGPU_DEEP_WARPS=6), c2 / c5 last 1000 MCS
run() { env $1 OCTGPU_DEEP_S=$2 timeout 300 python bench.py --config $4 --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/dw.json'));print('$4 $3 S=$2', round(d['roofline']['kernel_ms'],4), d.get('final_checksum'))"; }
D6=OCTGPU_LIB=tools/variants/dp6/liboctgpu.so
for rep in 1 2; do run "" 5 dp9 c2; run $D6 5 dp6 c2; run $D6 4 dp6 c2; run $D6 6 dp6 c2; done
run "" 5 dp9 c5; run $D6 5 dp6 c5
