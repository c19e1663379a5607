# k_mcs_bulk ring sweep (OCTGPU_MCS_KS x OCTGPU_MCS_S) at c3 / c2h from the flat start (profiles/r1_pipeline_sweep.json era)
for ks in 1 2 4; do for s in 2 3 4 6; do
OCTGPU_MCS_KS=$ks OCTGPU_MCS_S=$s timeout 120 python bench.py --config c3 --steps 200 --warmup 5 --from-flat --no-e2e --no-cpu-baseline > gpurun_out/sw_$ks.$s.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sw_$ks.$s.json'));print('c3 KS=$ks S=$s', round(d['roofline']['kernel_ms'],4), round(d['value']))"
done; done
for c in c2h; do for ks in 1 2 4; do for s in 2 3 4; do
OCTGPU_DEEP=0 OCTGPU_MCS_KS=$ks OCTGPU_MCS_S=$s timeout 120 python bench.py --config $c --steps 200 --warmup 5 --from-flat --no-e2e --no-cpu-baseline > gpurun_out/sw_$c$ks.$s.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sw_$c$ks.$s.json'));print('$c bulk KS=$ks S=$s', round(d['roofline']['kernel_ms'],4), round(d['value']))"
done; done; done
