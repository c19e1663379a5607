# k_mcs_deep (OCTGPU_DEEP=2) vs k_mcs_bulk (OCTGPU_DEEP=0) per live config, in the job's final window and from flat
for c in c3 c2h; do for dp in 0 2; do for ff in "" "--from-flat"; do
  OCTGPU_DEEP=$dp timeout 300 python bench.py --config $c --steps 1000 --warmup 3 $ff --no-e2e --no-cpu-baseline > gpurun_out/dvb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/dvb.json'));print('$c deep=$dp ${ff:-window}', round(d['roofline']['kernel_ms'],4), d['roofline']['kernel'])"
done; done; done
