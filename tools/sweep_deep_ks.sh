# k_mcs_deep words per ring stage (OCTGPU_DEEP_KS variants) x ring depth (OCTGPU_DEEP_S), c2 last 1000 MCS,
# (run while the default was OCTGPU_DEEP_KS=2 / deep_S=3; the variants were built with tools/build_variant.sh NAME -DOCTGPU_DEEP_KS=1|4)
# interleaved repetitions (box-to-box and run-to-run spread is a few %)
run() { env $1 OCTGPU_DEEP_S=$2 timeout 300 python bench.py --config c2 --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dks.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/dks.json'));print('$3 S=$2', round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])"; }
for rep in 1 2 3; do
  run "" 3 ks2; run "" 2 ks2
  run OCTGPU_LIB=tools/variants/dks1/liboctgpu.so 4 ks1; run OCTGPU_LIB=tools/variants/dks1/liboctgpu.so 5 ks1
done
