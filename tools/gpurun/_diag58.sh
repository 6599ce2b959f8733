timeout 900 python bench.py > /tmp/b.json 2>/tmp/b.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('/tmp/b.json'))
print('value', round(d['value']/1e6,3), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3), d['config']['victim_policy'])
print([(b['budget_frac'], b['victim_policy'], round(b['ms_per_step'],2), b['expert_loads_per_step']) for b in d['memory_regime_zipf']['budgets']])
print([(b['budget_frac'], b['victim_policy'], round(b['ms_per_step'],2), b['expert_loads_per_step']) for b in d['expert_streaming']['budgets']])
PY
