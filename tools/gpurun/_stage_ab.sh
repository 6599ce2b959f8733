# Token-N FFN: split A/B operand rings (A stages / B stages) vs the shared 6-stage ring (old)
mkdir -p gpurun_out/st
cp paper_2310_18859_b200/_sida_b200.so ab_cur.so
for r in 1 2; do
for v in old s66 s85 s94; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  echo "== $v run $r"
  timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas
  timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas --tokens 131072
  timeout 120 python tools/ffn_probe.py --experts 8 --no-cublas
  timeout 120 python tools/ffn_probe.py --experts 256 --no-cublas --tokens 65536
done
done 2>&1 | tee gpurun_out/st/ab.txt
cp ab_cur.so paper_2310_18859_b200/_sida_b200.so
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/st/tests.txt 2>&1; echo kernels_tests=$?
tail -2 gpurun_out/st/tests.txt
SIDA_GEMM_PROF=1 timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas | tee gpurun_out/st/prof.txt
for v in old cur old cur; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/st/bench_$v.json 2> gpurun_out/st/bench_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/st/bench_$v.json').read().strip().splitlines()[-1])
print('bench $v', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('step_ms_median'))"
done
cp ab_cur.so paper_2310_18859_b200/_sida_b200.so
