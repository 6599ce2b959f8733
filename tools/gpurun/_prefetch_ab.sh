# A/B of the residual L2 prefetch (SIDA_RESID_PREFETCH bitmask) on the out-projection and the FFN
mkdir -p gpurun_out/pf
for r in 1 2 3; do
for m in 0 1 3; do
  echo "== mode $m run $r"
  SIDA_RESID_PREFETCH=$m timeout 120 python tools/proj_probe.py
  SIDA_RESID_PREFETCH=$m timeout 120 python tools/ffn_probe.py --experts 128
done
done > gpurun_out/pf/ab.txt 2>&1
for m in 0 3; do
  SIDA_RESID_PREFETCH=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/pf/bench_$m.json 2> gpurun_out/pf/bench_$m.err
done
cat gpurun_out/pf/ab.txt
python - <<'P'
import json
for m in (0,3):
    try:
        d=json.loads(open(f"gpurun_out/pf/bench_{m}.json").read().strip().splitlines()[-1])
        print(m, d["value"], d["ms_per_step"], d["e2e"]["value"])
    except Exception as e: print(m, "ERR", e)
P
