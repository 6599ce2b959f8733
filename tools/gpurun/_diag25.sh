timeout 900 python -m pytest tests/test_gpu_serving.py tests/test_gpu_pipeline_contracts.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-extras --no-cpu-baseline > /tmp/b.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/b.json')); print('bench', round(d['ms_per_step'],3), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), [round(v/1e6,3) for v in d['e2e']['runs_tokens_per_s']])"; done
bash tools/gpurun/_diag23.sh
