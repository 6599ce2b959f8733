"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `sida` from /root/reference/pkg/src, runs the reference's own
public API on seeded inputs and writes small .npz / .json fixtures next to
this file. Those fixtures travel with the repo; nothing on the GPU box
reads /root/reference. The oracle (`oracle/`) is checked against them by
tests/test_oracle_golden.py, and the GPU path is checked against both.

Weights: the reference model draws float64 weights from its `Rng`; the
fixtures use those draws rounded to bf16 (oracle.numkit.round_bf16), the
exact values the bf16 GPU model holds (SURVEY §8(c) parity protocol). The
sha256 of the *unrounded* draws is recorded so the oracle's init can be
pinned to the reference's RNG stream.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from sida import numkit as ref_numkit  # noqa: E402
from sida.moe import MoEConfig, MoEModel, SequenceBatch, model_forward  # noqa: E402
from sida.numkit import Rng  # noqa: E402
from sida.offload import (  # noqa: E402
    MemoryBudget,
    ResidencyState,
    apply_plan,
    ensure_layer_resident,
    plan_placement,
)
from sida.pipeline import serve_sida, serve_standard  # noqa: E402
from sida.predictor import (  # noqa: E402
    OracleHasher,
    PredictorConfig,
    PredictorNet,
    build_hash_table,
    hash_hit_rate,
)

from oracle.numkit import round_bf16  # noqa: E402


def digest(params: dict) -> str:
    h = hashlib.sha256()
    for name in params:
        h.update(name.encode())
        h.update(np.ascontiguousarray(params[name], dtype=np.float64).tobytes())
    return h.hexdigest()


def numkit_case():
    g = np.random.default_rng(123)
    rows = [g.normal(0, 2, n) for n in (1, 2, 3, 7, 32, 128, 511)]
    rows.append(np.array([1.1, 1.0, -5.0]))
    rows.append(np.array([0.3, 0.3, 0.3, 0.3]))
    out = {}
    for i, r in enumerate(rows):
        out[f"sparsemax_in_{i}"] = r
        out[f"sparsemax_out_{i}"] = ref_numkit.sparsemax(r[None])[0]
        out[f"softmax_out_{i}"] = ref_numkit.softmax(r)
        kk = min(3, r.size)
        out[f"topk_out_{i}"] = ref_numkit.topk(r, kk)
    ties = np.array([[0.5, 0.7, 0.7, 0.1, 0.7], [1.0, 1.0, 1.0, 1.0, 1.0]])
    out["ties_in"] = ties
    out["ties_top3"] = ref_numkit.topk_rows(ties, 3)
    x = g.normal(0, 3, 64)
    out["sigmoid_in"] = x
    out["sigmoid_out"] = ref_numkit.sigmoid(x)
    np.savez_compressed(os.path.join(HERE, "numkit.npz"), **out)


def model_case(name, cfg, lengths, ks, pred_kwargs=None, seq_seed=2):
    model = MoEModel(cfg, Rng(0))
    raw_digest = digest(model.params)
    for k in model.params:
        model.params[k] = round_bf16(model.params[k])
    pcfg = PredictorConfig(**(pred_kwargs or {}))
    net = PredictorNet(pcfg, cfg.d_model, cfg.num_layers, cfg.num_experts, Rng(1))
    pred_digest = digest(net.params)
    rng = Rng(seq_seed)
    seqs = [rng.integers(0, cfg.vocab_size, size=n) for n in lengths]
    batch = SequenceBatch(0, seqs)
    out = {"lengths": np.array(lengths), "tokens": np.concatenate(seqs)}
    meta = {"config": cfg.__dict__, "predictor": {"compress_dim": pcfg.compress_dim,
            "lstm_hidden": pcfg.lstm_hidden}, "moe_digest": raw_digest,
            "predictor_digest": pred_digest, "ks": list(ks)}
    # predictor logits of the first sequence (forward contract)
    out["pred_logits_seq0"] = net.forward(model.embed(seqs[0]))
    for k in ks:
        table = build_hash_table(net, batch, k, model.embed)
        out[f"ids_k{k}"] = table.ids
        out[f"alphas_k{k}"] = table.alphas
        logits, trace = model_forward(model, batch, mode="external", table=table)
        out[f"logits_k{k}"] = logits
        # A13 contract fixture: numpy's stable argsort on the ref's ids
        for layer in range(cfg.num_layers):
            flat = table.ids[layer].reshape(-1)
            out[f"perm_k{k}_l{layer}"] = np.argsort(flat, kind="stable")
            out[f"hist_k{k}_l{layer}"] = np.bincount(flat, minlength=cfg.num_experts)
        # isolated layer: feed the reference moe_apply a fixed layer input
        t0 = lengths[0]
        x = model.attention_mix(0, model.embed(seqs[0]))
        out[f"layer0_in_k{k}"] = x
        out[f"layer0_out_k{k}"] = model.moe_apply(0, x, table.ids[0, :t0], table.alphas[0, :t0])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


class _Table:
    def __init__(self, layers):
        self.layers = [set(s) for s in layers]

    def required_by_layer(self):
        return self.layers

    def required_experts(self):
        return {(l, e) for l, s in enumerate(self.layers) for e in s}


def planner_case():
    g = np.random.default_rng(7)
    cases = []
    eb = 1000
    for ci in range(40):
        n_layers = int(g.integers(1, 5))
        n_exp = int(g.integers(2, 9))
        slots = int(g.integers(1, n_layers * n_exp + 2))
        budget = MemoryBudget(slots * eb, bandwidth_bytes_per_s=1e6, per_transfer_latency_s=1e-3)
        state = ResidencyState()
        batches = []
        for _ in range(int(g.integers(1, 6))):
            req = [sorted(set(g.integers(0, n_exp, size=int(g.integers(1, n_exp + 1))).tolist()))
                   for _ in range(n_layers)]
            plan = plan_placement(_Table(req), state, budget, eb)
            state, secs = apply_plan(state, plan)
            batches.append({
                "required": req,
                "groups": [{"layer": gr.layer, "steps": [[op, list(k)] for op, k in gr.steps],
                            "prefetchable": gr.prefetchable, "transfer_s": gr.transfer_s}
                           for gr in plan.groups],
                "fifo_after": [list(k) for k in state.fifo_order],
                "seconds": secs,
            })
        cases.append({"slots": slots, "expert_bytes": eb, "bandwidth": 1e6, "latency": 1e-3,
                      "batches": batches})
    with open(os.path.join(HERE, "planner.json"), "w") as fh:
        json.dump(cases, fh)


def router_case(name, cfg, lengths, eval_ks, seq_seed=2):
    """Router mode (the teacher path): model_forward(mode="router"), the
    OracleHasher table, hash_hit_rate of the predictor's tables against the
    teacher traces, serve_standard with a tight budget and serve_sida with
    the oracle hasher (predictor=None)."""
    model = MoEModel(cfg, Rng(0))
    for k in model.params:
        model.params[k] = round_bf16(model.params[k])
    net = PredictorNet(PredictorConfig(), cfg.d_model, cfg.num_layers, cfg.num_experts, Rng(1))
    rng = Rng(seq_seed)
    seqs = [rng.integers(0, cfg.vocab_size, size=n) for n in lengths]
    batch = SequenceBatch(0, seqs)
    out = {"lengths": np.array(lengths), "tokens": np.concatenate(seqs)}
    logits, trace = model_forward(model, batch, mode="router")
    out["logits"] = logits
    out["selected"] = trace.selected
    out["alphas"] = trace.alphas
    out["probs"] = trace.probs
    # layer-0 router input (attention output of every sequence) for the kernel check
    out["router_in_l0"] = np.concatenate(
        [model.attention_mix(0, model.embed(s)) for s in seqs])
    for k in eval_ks:
        t = OracleHasher(model).build_table(batch, k)
        out[f"oracle_ids_k{k}"] = t.ids
        out[f"oracle_alphas_k{k}"] = t.alphas
        pt = build_hash_table(net, batch, k, model.embed)
        out[f"pred_ids_k{k}"] = pt.ids
        out[f"hit_rate_k{k}"] = np.array(hash_hit_rate([pt], [trace], k))
    eb = model.expert_bytes_each()
    budget = MemoryBudget(max(1, cfg.num_experts // 2) * eb)
    rep = serve_standard(model, [batch, SequenceBatch(1, seqs[::-1])], budget)
    out["standard_logits_b0"] = rep.logits[0]
    out["standard_logits_b1"] = rep.logits[1]
    out["standard_peak"] = np.array(rep.peak_fast_tier_bytes // eb)
    rep = serve_sida(model, None, [batch], MemoryBudget(cfg.num_layers * cfg.num_experts * eb),
                     eval_top_k=1)
    out["oracle_serve_hit_rate"] = np.array(rep.hit_rate)
    out["oracle_serve_logits"] = rep.logits[0]
    np.savez_compressed(os.path.join(HERE, f"router_{name}.npz"), **out)


def ensure_case():
    """ensure_layer_resident (ref offload.py:240-278) on random request streams."""
    g = np.random.default_rng(11)
    cases = []
    eb = 1000
    for _ in range(40):
        n_layers, n_exp = int(g.integers(1, 5)), int(g.integers(2, 9))
        slots = int(g.integers(1, n_layers * n_exp + 2))
        budget = MemoryBudget(slots * eb)
        state = ResidencyState()
        calls = []
        for _ in range(int(g.integers(1, 12))):
            layer = int(g.integers(0, n_layers))
            req = sorted(set(g.integers(0, n_exp, size=int(g.integers(1, n_exp + 1))).tolist()))
            grp = ensure_layer_resident(state, layer, req, budget, eb)
            calls.append({"layer": layer, "required": req,
                          "steps": [[op, list(k)] for op, k in grp.steps],
                          "transfer_s": grp.transfer_s,
                          "fifo_after": [list(k) for k in state.fifo_order]})
        cases.append({"slots": slots, "expert_bytes": eb, "calls": calls})
    with open(os.path.join(HERE, "ensure.json"), "w") as fh:
        json.dump(cases, fh)


def checkpoint_case():
    """Reference-written containers (ref checkpoint.py, moe.py:581-596,
    predictor.py:550-571): a small tcgen05-shaped model and its predictor."""
    from sida.moe import save_moe
    from sida.predictor import save_predictor

    cfg = MoEConfig(vocab_size=64, d_model=64, num_layers=2, num_experts=4, expert_hidden=128,
                    max_seq_len=16, routing_k=1, num_classes=3)
    save_moe(MoEModel(cfg, Rng(0)), os.path.join(HERE, "mini64.sidamoe"))
    net = PredictorNet(PredictorConfig(compress_dim=8, lstm_hidden=16), cfg.d_model,
                       cfg.num_layers, cfg.num_experts, Rng(1))
    save_predictor(net, os.path.join(HERE, "mini64.sidahsh"))


def main():
    if "--checkpoint" in sys.argv:  # container fixtures only
        checkpoint_case()
        return
    if "--router" in sys.argv:  # router-mode fixtures only (added after the first set)
        router_main()
        return
    numkit_case()
    model_case("tiny", MoEConfig(vocab_size=64, d_model=32, num_layers=2, num_experts=8,
                                 expert_hidden=64, max_seq_len=16, routing_k=1, num_classes=3),
               lengths=[5, 16, 9, 1, 12], ks=(1, 2, 3))
    # C0 of BASELINE.json: 2 MoE layers, 8 experts, d=256, top-1, 8x128 tokens
    model_case("c0", MoEConfig(vocab_size=512, d_model=256, num_layers=2, num_experts=8,
                               expert_hidden=1024, max_seq_len=128, routing_k=1, num_classes=4),
               lengths=[128] * 8, ks=(1,))
    planner_case()
    router_main()
    checkpoint_case()


def router_main():
    router_case("tiny", MoEConfig(vocab_size=64, d_model=32, num_layers=2, num_experts=8,
                                  expert_hidden=64, max_seq_len=16, routing_k=1, num_classes=3),
                lengths=[5, 16, 9, 1, 12], eval_ks=(1, 2))
    router_case("tiny_r2", MoEConfig(vocab_size=64, d_model=32, num_layers=3, num_experts=6,
                                     expert_hidden=64, max_seq_len=16, routing_k=2,
                                     num_classes=3),
                lengths=[7, 16, 3], eval_ks=(1, 3))
    router_case("c0", MoEConfig(vocab_size=512, d_model=256, num_layers=2, num_experts=8,
                                expert_hidden=1024, max_seq_len=128, routing_k=1, num_classes=4),
                lengths=[128] * 8, eval_ks=(1,))
    ensure_case()


if __name__ == "__main__":
    main()
