# L2 prefetch distance (OCTGPU_PREFETCH, ring stages) with the one-word deep ring, c2 last 1000 MCS, interleaved
for rep in 1 2; do for pf in 0 4 8 16; do
  OCTGPU_PREFETCH=$pf timeout 300 python bench.py --config c2 --steps 1000 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pf.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pf.json'));print('pf=$pf', round(d['roofline']['kernel_ms'],4))"
done; done
