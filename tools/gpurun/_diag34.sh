SIDA_GEMM_PROF=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas 2>&1 | head -8
for i in 1 2; do timeout 600 python bench.py --no-extras --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err; python -c "import json; d=json.load(open('/tmp/b.json')); r=d['roofline']; print('bench', round(d['ms_per_step'],3), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'ffn', round(r['avg_ms'],4), 'frac', round(r['frac'],3), 'mhz', r['ffn_kernel_sm_mhz'], 'mix', round(r['attention_mix_avg_ms'],4))"; done
tail -3 /tmp/b.err
