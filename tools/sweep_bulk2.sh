# k_mcs_bulk ring (OCTGPU_MCS_KS x OCTGPU_MCS_S) for the configs it serves, last 1000 MCS (c4: 30 from flat),
# interleaved repetitions
run() { OCTGPU_MCS_KS=$1 OCTGPU_MCS_S=$2 timeout 300 python bench.py --config $3 $4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b2.json'));print('$3 KS=$1 S=$2', round(d['roofline']['kernel_ms'],4))"; }
for rep in 1 2; do
  for ks_s in "2 2" "1 3" "1 4" "1 5" "2 3"; do set -- $ks_s; run $1 $2 c3 "--steps 1000"; done
done
for ks_s in "2 2" "1 3" "1 4" "1 5"; do set -- $ks_s; run $1 $2 c4 "--steps 30"; done
