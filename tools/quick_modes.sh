# kernel ms/MCS and final checksums for the live configs (bench --from-flat, short runs)
TAG=${1:-q}
for c in c2h c3 c4; do
  S=200; [ $c = c4 ] && S=20
  timeout 300 python bench.py --config $c --steps $S --warmup 3 --from-flat --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$c.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_$c.json'));print('$c', round(d['roofline']['kernel_ms'],4), d['roofline']['kernel'], d.get('final_checksum'))"
done
