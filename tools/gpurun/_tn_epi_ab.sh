# token-N GEMM2 epilogue: residual rows one chunk ahead vs per chunk (old)
mkdir -p gpurun_out/tne
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/tne/tests.txt 2>&1; echo tests=$?
tail -2 gpurun_out/tne/tests.txt
for r in 1 2 3; do
for v in old new; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  echo "== $v run $r"
  timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas
  timeout 120 python tools/ffn_probe.py --experts 8 --no-cublas
  timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas --tokens 131072
done
done 2>&1 | tee gpurun_out/tne/ab.txt
for v in old new old new; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/tne/bench_$v.json 2> gpurun_out/tne/bench_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/tne/bench_$v.json').read().strip().splitlines()[-1])
print('bench $v', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('step_ms_median'))"
done
cp ab_new.so paper_2310_18859_b200/_sida_b200.so
