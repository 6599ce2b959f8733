mkdir -p gpurun_out/d55
timeout 900 python bench.py > gpurun_out/d55/bench.json 2> gpurun_out/d55/bench.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/d55/bench.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['runs_tokens_per_s'])
r=d['roofline']; print({k: r[k] for k in ('frac','peak','frac_vs_burst_peak','ffn_kernel_sm_mhz','avg_ms','attention_mix_avg_ms','share_of_step')})
for s in d['north_star_ffn']['shapes']+[d['north_star_ffn']['balanced_base8']]: print({k: s[k] for k in ('experts','tokens','avg_ms','frac','kernel_sm_mhz','frac_vs_burst_peak')})
print(d['clocks'])
print(d['rooflines']['hash'])
for b in d['expert_streaming']['budgets']: print('stream', b['budget_frac'], b['victim_policy'], round(b['ms_per_step'],3), round(b['exposed_ms_per_step'],3))
for b in d['memory_regime_zipf']['budgets']: print('zipf', b['budget_frac'], round(b['ms_per_step'],3), round(b['exposed_ms_per_step'],3), round(b['memory_reduction_per_batch'],3))
PY
