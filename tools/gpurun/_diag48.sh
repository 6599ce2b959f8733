for cfg in "X=0" "SIDA_XBATCH_LOOKAHEAD=2" "SIDA_XBATCH_LOOKAHEAD=4" "SIDA_PREFETCH_DEPTH=3" "SIDA_PREFETCH_DEPTH=6" "SIDA_XBATCH_LOOKAHEAD=3 SIDA_PREFETCH_DEPTH=3"; do
  for bf in 0.97 0.9; do env $cfg timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 --budget-frac $bf > /tmp/b.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/b.json')); print('$cfg bf $bf', round(d['ms_per_step'],3), 'med', round(d['step_ms_median'],3), 'loads/step', d['expert_memory']['expert_loads_timed_region']/20)"; done
done
