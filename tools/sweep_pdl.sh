# programmatic dependent launch of k_mcs_deep (OCTGPU_PDL=0/1), c2 / c2h / c5 last 1000 MCS, interleaved
# (the OCTGPU_PDL launch path was removed after this measurement)
run() { OCTGPU_PDL=$1 timeout 300 python bench.py --config $2 --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pdl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pdl.json'));print('$2 pdl=$1', round(d['roofline']['kernel_ms'],4), round(d['value']), d.get('final_checksum'))"; }
for rep in 1 2; do run 0 c2; run 1 c2; done
for c in c2h c5; do run 0 $c; run 1 $c; done
