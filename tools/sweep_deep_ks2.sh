# k_mcs_deep KS=1 ring depths vs the KS=2 default, c2 / c2h / c5 (last 1000 MCS), interleaved
# (run while the default was OCTGPU_DEEP_KS=2 / deep_S=3; the variants were built with tools/build_variant.sh NAME -DOCTGPU_DEEP_KS=1|4)
run() { env $1 OCTGPU_DEEP_S=$2 timeout 300 python bench.py --config $4 --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dks.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/dks.json'));print('$4 $3 S=$2', round(d['roofline']['kernel_ms'],4), d.get('final_checksum'))"; }
K1=OCTGPU_LIB=tools/variants/dks1/liboctgpu.so
for rep in 1 2; do
  run "" 3 ks2 c2; run $K1 5 ks1 c2; run $K1 6 ks1 c2; run $K1 7 ks1 c2
done
for c in c2h c5; do run "" 3 ks2 $c; run $K1 5 ks1 $c; run $K1 6 ks1 $c; done
