mkdir -p gpurun_out/h2
for A in 1 2; do timeout 300 python tools/host_time.py --experts 128 --budget-frac 0.97 --ahead $A; done > gpurun_out/h2/host.txt 2>&1
timeout 300 python tools/host_time.py --experts 128 --budget-frac 0.97 --ahead 2 --profile > gpurun_out/h2/prof.txt 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/h2/bench.json 2> gpurun_out/h2/bench.err
cat gpurun_out/h2/host.txt; head -60 gpurun_out/h2/prof.txt | cut -c1-150; python -c "import json; d=json.load(open('gpurun_out/h2/bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['avg_ms'], d['roofline']['attention_mix_avg_ms'], d['clocks'])"
