for GC_OFF in 0 1; do export GC_OFF; echo GC_OFF=$GC_OFF; timeout 900 python - <<'PY'
import sys, json, os, time
sys.argv=['bench.py']
sys.path.insert(0, '.')
import bench, torch, numpy as np
from paper_2310_18859_b200 import MoEConfig, MoEModel, PredictorConfig, PredictorNet, Rng, MemoryBudget
from paper_2310_18859_b200.engine import SidaEngine
cfg = MoEConfig(**dict(bench.SWITCH, num_experts=128))
model = MoEModel.synthetic(cfg, seed=0)
pred = PredictorNet(PredictorConfig(), cfg.d_model, cfg.num_layers, cfg.num_experts, Rng(1))
lengths=[128]*256
n_tok=sum(lengths)
g = torch.Generator(device=model.device); g.manual_seed(4321)
toks = [bench.synth_tokens(n_tok, cfg.vocab_size, g) for _ in range(7)]
eb = model.expert_bytes_each()
import gc
GC = os.environ.get("GC_OFF") == "1"
if GC: gc.collect(); gc.freeze(); gc.disable()
for rep in range(3):
    for frac in (1.0, 0.9):
        slots = int(round(frac * 1536))
        eng = SidaEngine(model, pred, MemoryBudget(slots * eb), eval_top_k=1, victim_policy="spread")
        bench.run_stream(eng, toks, lengths, 3, 1)
        cs = eng.compute_stream
        tables = {i: eng.hash_tokens(i, toks[i], lengths) for i in range(2)}
        evs=[]
        torch.cuda.synchronize()
        t0=time.perf_counter()
        for j in range(6):
            e=torch.cuda.Event(enable_timing=True); e.record(cs); evs.append(e)
            a=j+2
            tables[a]=eng.hash_tokens(a, toks[a%7], lengths)
            eng.forward(tables.pop(j), lengths, tokens_dev=toks[j%7], next_table=tables[j+1])
        e=torch.cuda.Event(enable_timing=True); e.record(cs); evs.append(e)
        torch.cuda.synchronize()
        print(rep, frac, [round(evs[i].elapsed_time(evs[i+1]),2) for i in range(6)], 'host', round((time.perf_counter()-t0)*1e3,1), 'loads', eng.store.n_loads, flush=True)
        del eng, tables
        torch.cuda.empty_cache()
PY
done
