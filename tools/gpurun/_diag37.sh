timeout 900 python - <<'PY'
import sys, json, os
sys.argv=['bench.py']
sys.path.insert(0, '.')
import bench, torch, numpy as np
from paper_2310_18859_b200 import MoEConfig, MoEModel, PredictorConfig, PredictorNet, Rng
cfg = MoEConfig(**dict(bench.SWITCH, num_experts=128))
model = MoEModel.synthetic(cfg, seed=0)
pred = PredictorNet(PredictorConfig(), cfg.d_model, cfg.num_layers, cfg.num_experts, Rng(1))
lengths=[128]*256
for rep in range(2):
    out = bench.budget_runs(model, pred, cfg, lengths, [(1.0, "fifo"), (0.97, "spread"), (0.97, "fifo"), (0.9, "spread"), (0.75, "spread")])
    for b in out: print(rep, b['budget_frac'], b['victim_policy'], round(b['ms_per_step'],3), round(b['exposed_ms_per_step'],3), round(b['expert_loads_per_step'],2))
PY
