mkdir -p gpurun_out/d16
timeout 900 python bench.py > gpurun_out/d16/bench.json 2> gpurun_out/d16/bench.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/d16/bench.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'])
r=d['roofline']; print({k: r[k] for k in ('frac','peak','peak_source','frac_vs_burst_peak','ffn_kernel_sm_mhz','avg_ms','attention_mix_avg_ms')})
for s in d['north_star_ffn']['shapes']+[d['north_star_ffn']['balanced_base8']]: print({k: s[k] for k in ('experts','tokens','avg_ms','frac','kernel_sm_mhz','frac_vs_burst_peak')})
print(d['clocks'])
print(d['rooflines']['permute_c4_scale'], d['rooflines']['permute_bench_scale'])
PY
tail -3 gpurun_out/d16/bench.err
