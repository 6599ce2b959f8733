mkdir -p gpurun_out/ser
for s in "" 1 "" 1; do
  SIDA_HASH_SERIAL=$s timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ser/bench_$s.json 2> gpurun_out/ser/bench_$s.err
  python -c "
import json
d=json.loads(open('gpurun_out/ser/bench_$s.json').read().strip().splitlines()[-1])
print('bench serial=$s', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('step_ms_median'))"
done
