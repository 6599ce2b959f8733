# token-M STAGE-2 epilogue (attention output projection): residual loads one chunk ahead vs per chunk
mkdir -p gpurun_out/epi
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 600 -p no:cacheprovider -k "out_proj or grouped_ffn_bf16 or token_n" > gpurun_out/epi/tests.txt 2>&1; echo kernels_tests=$?
tail -2 gpurun_out/epi/tests.txt
for r in 1 2 3; do
for v in old new; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  echo "== $v run $r"
  timeout 120 python tools/proj_probe.py
  SIDA_FFN_SWAP=0 timeout 120 python tools/ffn_probe.py --experts 8 --no-cublas
done
done 2>&1 | tee gpurun_out/epi/ab.txt
for v in old new old new; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/epi/bench_$v.json 2> gpurun_out/epi/bench_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/epi/bench_$v.json').read().strip().splitlines()[-1])
print('bench $v', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('step_ms_median'))"
done
cp ab_new.so paper_2310_18859_b200/_sida_b200.so
