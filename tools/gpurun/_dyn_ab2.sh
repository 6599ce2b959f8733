# Ticket schedule (drawn one tile ahead) vs static, and the LPT token-tile order, token-N FFN GEMMs
mkdir -p gpurun_out/dyn2
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 600 -p no:cacheprovider -k "ticket or token_n or grouped_ffn_bf16" > gpurun_out/dyn2/tests.txt 2>&1; echo kernels_tests=$?
tail -3 gpurun_out/dyn2/tests.txt
for r in 1 2; do
for cfg in "0 0" "0 1" "1 1"; do
  set -- $cfg
  echo "== dyn $1 lpt $2 run $r"
  SIDA_DYN_SCHED=$1 SIDA_TN_LPT=$2 timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas
  SIDA_DYN_SCHED=$1 SIDA_TN_LPT=$2 timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas --tokens 131072
  SIDA_DYN_SCHED=$1 SIDA_TN_LPT=$2 timeout 120 python tools/ffn_probe.py --experts 8 --no-cublas
done
done 2>&1 | tee gpurun_out/dyn2/ab.txt
SIDA_GEMM_PROF=1 timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas | tee gpurun_out/dyn2/prof.txt
for m in 0 1 0 1; do
  SIDA_DYN_SCHED=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/dyn2/bench_$m.json 2> gpurun_out/dyn2/bench_$m.err
  python -c "
import json
d=json.loads(open('gpurun_out/dyn2/bench_$m.json').read().strip().splitlines()[-1])
print('bench dyn=$m', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('step_ms_median'))"
done
