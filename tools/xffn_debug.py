"""One-launch expert FFN determinism probe: full launch vs repeated full
launch vs expert-list waves, max |diff| and the experts whose rows differ."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import _lib  # noqa: E402
from paper_2310_18859_b200.moe import MoEConfig, MoEModel  # noqa: E402
from paper_2310_18859_b200.offload import ExpertStore, Wave, run_waves  # noqa: E402
from paper_2310_18859_b200.predictor import ExpertHashTable  # noqa: E402

h = _lib.load()
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 5
_lib.check(h.sida_set_ffn_tiles(mode))
d, hd, K, N = 256, 1024, 8, 3000
cfg = MoEConfig(vocab_size=64, d_model=d, num_layers=1, num_experts=K, expert_hidden=hd,
                max_seq_len=16)
model = MoEModel.synthetic(cfg, 0)
g = np.random.default_rng(11)
ids = g.integers(0, K, size=(1, N, 1))
al = g.uniform(0.05, 1.0, size=ids.shape)
dt = ExpertHashTable(0, [N], ids, al).on_device(model)
x = torch.from_numpy(g.normal(0, 1.0, (N, d))).float().cuda()
store = ExpertStore.full(model)
st = torch.cuda.current_stream()
store.run_layer(model, 0, x, dt)  # loads every expert of the layer
torch.cuda.synchronize()
row = store.slot_row(0, list(range(K)))
outs = [run_waves(model, [Wave(0, [], list(range(K)), row)], x, dt, store, st) for _ in range(3)]
outs.append(run_waves(model, [Wave(0, [], [0, 2, 4, 6], row), Wave(0, [], [1, 3, 5, 7], row)],
                      x, dt, store, st))
outs.append(run_waves(model, [Wave(0, [], [1, 3, 5, 7], row), Wave(0, [], [0, 2, 4, 6], row)],
                      x, dt, store, st))
torch.cuda.synchronize()
print("nan rows per run:", [int(torch.isnan(o).any(1).sum()) for o in outs],
      "x nan:", bool(torch.isnan(x).any()))
nanrows = torch.nonzero(torch.isnan(outs[0]).any(1)).flatten().cpu().numpy()
print("experts of nan rows:", sorted(set(ids[0, nanrows, 0].tolist())), "count", len(nanrows))
for i, o in enumerate(outs[1:], 1):
    dif = (o - outs[0]).abs()
    rows = torch.nonzero(dif.amax(1) > 0).flatten().cpu().numpy()
    print(f"run {i}: max diff {dif.max().item():.3e}, rows differing {len(rows)}, experts "
          f"{sorted(set(ids[0, rows, 0].tolist()))[:8]}")
