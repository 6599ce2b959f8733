timeout 900 python - <<'PY'
import sys, os, time, gc
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
eb = model.expert_bytes_each()
eng = SidaEngine(model, pred, MemoryBudget(1490 * eb), eval_top_k=1, victim_policy="spread")
g = torch.Generator(device=model.device); g.manual_seed(1234)
toks14 = [bench.synth_tokens(n_tok, cfg.vocab_size, g) for _ in range(14)]
gc.collect(); gc.freeze()
for rep in range(3):
    ms, _ = bench.run_stream(eng, toks14, lengths, 10, 3)
    ms9, _ = bench.run_stream(eng, toks14[:9], lengths, 6, 2)
    print(rep, 'run_stream 14 toks median', round(ms,3), '| 9 toks median', round(ms9,3), flush=True)
PY
