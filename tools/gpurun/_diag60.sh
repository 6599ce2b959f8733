set -x
timeout 300 python -m pytest tests -q -m gpu -k "permute or route or hash or parity or smoke" -x 2>&1 | tail -3
for a in "--rows 262144 --experts 256" "--rows 32768 --experts 128" "--rows 32768 --experts 8" "--rows 131072 --experts 128"; do timeout 120 python tools/permute_probe.py --layers 12 $a; done
for r in 1 2; do timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 > /tmp/b.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/b.json')); print(round(d['ms_per_step'],3), 'med', round(d['step_ms_median'],3), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'ffn', round(d['roofline']['avg_ms'],4))"; done
