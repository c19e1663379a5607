# counter-based rng mode (bench --rng counter, k_sweep_ctr) per config, short runs from the flat start
for c in c2 c2h c3 c4; do
  S=200; [ $c = c4 ] && S=20
  timeout 300 python bench.py --config $c --rng counter --steps $S --warmup 3 --from-flat --no-e2e --no-cpu-baseline > gpurun_out/ctr_$c.json
  python -c "import json;d=json.load(open('gpurun_out/ctr_$c.json'));print('$c', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), d.get('final_checksum'))"
done
