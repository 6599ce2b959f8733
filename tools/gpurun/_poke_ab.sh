# HEAD (pinned H2D small rows, tokens uploaded inside the hash) vs this tree (sida_poke_i32 rows, tokens pre-uploaded)
mkdir -p gpurun_out/poke
swap() { for f in pipeline.py predictor.py offload.py _lib.py _sida_b200.so; do cp abset/$1/$f paper_2310_18859_b200/$f; done; }
for r in 1 2; do
for v in old new; do
  swap $v
  timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/poke/bench_$v.json 2> gpurun_out/poke/bench_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/poke/bench_$v.json').read().strip().splitlines()[-1])
print('bench $v', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('step_ms_median'))"
  echo "== e2e probe $v"; timeout 300 python tools/e2e_probe.py --batches 20 --reps 2 2>&1 | grep "^rep"
done
done 2>&1 | tee gpurun_out/poke/ab.txt
swap new
SIDA_HASH_SERIAL=1 timeout 300 python tools/serial_probe.py 2>&1 | tee gpurun_out/poke/timeline_serial.txt
SIDA_HASH_SERIAL=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench new serial', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']))"
