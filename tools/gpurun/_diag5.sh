mkdir -p gpurun_out/d5
{
for i in 1 2; do timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 > gpurun_out/d5/b$i.json 2>gpurun_out/d5/b$i.err; python -c "import json; d=json.load(open('gpurun_out/d5/b$i.json')); print('bench', round(d['value']/1e6,3), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3), 'ffn', round(d['roofline']['avg_ms'],3), 'mix', round(d['roofline']['attention_mix_avg_ms'],3), d['clocks']['sm_mhz'])"; done
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 --budget-frac 1.0 > gpurun_out/d5/bfull.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/d5/bfull.json')); print('bench full budget', round(d['value']/1e6,3), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3))"
echo "== CG2 both"; SIDA_FFN_CG=2 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== CG1 both"; SIDA_FFN_CG=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== BN2=192"; SIDA_FFN_BN2=192 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== PDL off"; SIDA_PDL=0 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
} > gpurun_out/d5/out.txt 2>&1
cat gpurun_out/d5/out.txt
