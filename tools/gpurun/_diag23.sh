python tools/pipe_ab.py --modes flat,serial --reps 3 --steps 10 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-extras --no-cpu-baseline --budget-frac 1.0 --steps 10 > /tmp/b.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/b.json')); print('bench full', round(d['ms_per_step'],3), round(d['value']/1e6,3))"; done
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 10 > /tmp/b.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/b.json')); print('bench 0.97', round(d['ms_per_step'],3), round(d['value']/1e6,3))"
