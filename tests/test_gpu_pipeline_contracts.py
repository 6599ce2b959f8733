"""Serving contracts of the reference's tests/test_pipeline.py on the GPU
path, on small tcgen05-shaped models (d=64, h=128; the reference uses d=16,
below the tensor-core tile): oracle-vs-standard equivalence, the full-width
table against dense soft routing, determinism, the per-batch breakdown and
the report files."""

import json

import numpy as np
import pytest

from oracle import moe as omoe
from oracle import numkit as onk
from oracle import predictor as opred
from test_gpu_kernels import close_rms

pytestmark = pytest.mark.gpu

BASE = dict(vocab_size=32, d_model=64, num_layers=2, num_experts=4, expert_hidden=128,
            max_seq_len=12, routing_k=1, num_classes=3)


def make_model(seed=0):
    from paper_2310_18859_b200 import MoEConfig, MoEModel, Rng

    return MoEModel(MoEConfig(**BASE), Rng(seed))


def make_stream(model, n_batches, seed=0, batch_size=3, t_len=(4, 9)):
    from paper_2310_18859_b200 import Rng, SequenceBatch

    rng = Rng(seed)
    out = []
    for i in range(n_batches):
        seqs = [rng.integers(0, model.config.vocab_size, size=int(rng.integers(*t_len)))
                for _ in range(batch_size)]
        labels = [int(rng.integers(0, model.config.num_classes)) for _ in seqs]
        out.append(SequenceBatch(i, seqs, labels))
    return out


def unlimited(model):
    from paper_2310_18859_b200 import MemoryBudget

    return MemoryBudget(model.total_expert_bytes())


def test_sida_oracle_matches_standard(cuda_device):
    """ref test_pipeline.py:74-83: the teacher routers as hash function serve
    the same logits as router-mode standard serving; hit rate 1, fidelity 1."""
    from paper_2310_18859_b200 import fidelity, serve_sida, serve_standard

    model = make_model(3)
    stream = make_stream(model, 6, seed=5)
    ro = serve_sida(model, None, stream, unlimited(model), eval_top_k=1)
    rs = serve_standard(model, stream, unlimited(model))
    assert ro.mode == "oracle" and rs.mode == "standard"
    assert len(ro.logits) == len(rs.logits) == 6
    for a, b in zip(ro.logits, rs.logits):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)
    assert fidelity(ro, rs) == 1.0
    assert ro.hit_rate == 1.0


def test_single_batch_stream(cuda_device):
    from paper_2310_18859_b200 import serve_sida

    model = make_model(4)
    rep = serve_sida(model, None, make_stream(model, 1, seed=6), unlimited(model), eval_top_k=1)
    assert len(rep.batch_records) == 1
    assert rep.batch_records[0]["queue_wait_s"] >= 0.0


def test_full_width_table_matches_dense_soft_routing(cuda_device):
    """ref test_pipeline.py:92-123: eval_top_k = K with an unlimited budget is
    the dense alpha-weighted sum over all experts, alpha = the predictor's
    full softmax (k = K > 4 also exercises the gather + rank-combine path)."""
    from paper_2310_18859_b200 import PredictorConfig, PredictorNet, serve_sida

    model = make_model(7)
    K, L = BASE["num_experts"], BASE["num_layers"]
    pp = opred.init_params(opred.PredictorShape(64, L, K, compress_dim=6, lstm_hidden=8), 9)
    pred = PredictorNet(PredictorConfig(compress_dim=6, lstm_hidden=8, top_t=2), 64, L, K,
                        params=pp)
    stream = make_stream(model, 3, seed=8)
    rep = serve_sida(model, pred, stream, unlimited(model), eval_top_k=K, compute_hit_rate=False)
    shape = omoe.MoEShape(**BASE)
    params = omoe.bf16_params(omoe.init_params(shape, 7))
    for batch, logits in zip(stream, rep.logits):
        for si, tokens in enumerate(batch.sequences):
            emb = omoe.embed(params, shape, tokens)
            probs = onk.softmax(opred.forward(pp, emb))
            x = emb
            for layer in range(L):
                x = omoe.attention_mix(params, shape, layer, x)
                pre = f"block{layer}."
                out = np.zeros_like(x)
                for e in range(K):
                    hid = np.maximum(x @ params[pre + "w1"][e] + params[pre + "b1"][e], 0.0)
                    out += probs[layer][:, e][:, None] * (hid @ params[pre + "w2"][e]
                                                          + params[pre + "b2"][e])
                x = x + out
            close_rms(logits[si], x.mean(axis=0) @ params["wc"], 2e-2)


def test_five_runs_bitwise_identical_logits(cuda_device):
    """ref test_pipeline.py:127-142 (tight budget: reactive loads every layer)."""
    from paper_2310_18859_b200 import MemoryBudget, serve_standard

    model = make_model(11)
    stream = make_stream(model, 5, seed=12)
    budget = MemoryBudget(2 * model.expert_bytes_each())
    runs = [serve_standard(model, stream, budget) for _ in range(5)]
    for r in runs[1:]:
        for a, b in zip(runs[0].logits, r.logits):
            np.testing.assert_array_equal(a, b)
    assert runs[0].peak_fast_tier_bytes <= 2 * model.expert_bytes_each()


def test_breakdown_fields_present(cuda_device):
    """ref test_pipeline.py:203-212."""
    from paper_2310_18859_b200 import serve_standard

    model = make_model(21)
    rep = serve_standard(model, make_stream(model, 3, seed=22), unlimited(model),
                         selection_overhead_s=1e-3)
    for rec in rep.batch_records:
        assert rec["selection_s"] >= 1e-3 * model.config.num_layers
        assert rec["compute_s"] > 0.0
        assert "transfer_s" in rec and "latency_s" in rec


def test_report_json_and_csv_from_a_run(cuda_device, tmp_path):
    """ref test_pipeline.py:257-270."""
    from paper_2310_18859_b200 import serve_sida

    model = make_model(25)
    rep = serve_sida(model, None, make_stream(model, 4, seed=26), unlimited(model), eval_top_k=1)
    rep.save_json(tmp_path / "report.json")
    rep.save_csv(tmp_path / "report.csv")
    data = json.loads((tmp_path / "report.json").read_text())
    assert data["schema_version"] == 1
    assert len(data["batches"]) == 4
    assert data["aggregate"]["throughput_samples_per_s"] > 0
    assert data["aggregate"]["hash_hit_rate"] == 1.0


def test_engine_ring_reused_across_calls_and_after_a_failed_call(cuda_device):
    """serve_sida keeps its device table ring (and pinned token staging) with
    the engine: repeated calls over the same batches give identical logits,
    and a call that raises mid-stream (a token outside the vocabulary in its
    third batch) leaves the engine serving correctly afterwards."""
    from paper_2310_18859_b200 import (ContractError, MemoryBudget, PredictorConfig,
                                       PredictorNet, Rng, SequenceBatch, serve_sida)
    from paper_2310_18859_b200.engine import SidaEngine

    model = make_model()
    pred = PredictorNet(PredictorConfig(), BASE["d_model"], BASE["num_layers"],
                        BASE["num_experts"], Rng(1))
    budget = MemoryBudget(3 * model.expert_bytes_each())
    eng = SidaEngine(model, pred, budget)
    batches = make_stream(model, 5)
    runs = [serve_sida(model, pred, batches, budget, engine=eng, compute_hit_rate=False)
            for _ in range(2)]
    assert eng._serve_ring is not None
    bad = list(batches)
    bad[2] = SequenceBatch(2, [np.array([0, BASE["vocab_size"]])])
    with pytest.raises(ContractError):
        serve_sida(model, pred, bad, budget, engine=eng, compute_hit_rate=False)
    runs.append(serve_sida(model, pred, batches, budget, engine=eng, compute_hit_rate=False))
    for r in runs[1:]:
        for a, b in zip(runs[0].logits, r.logits):
            assert np.array_equal(a, b)


def test_engine_token_pool_grows_across_calls(cuda_device):
    """serve_sida's per-engine token pool (tokens uploaded one iteration ahead
    on their own stream, SM-copied from pinned staging) is reallocated when a
    later call brings larger batches and reused when it brings smaller ones:
    every call matches a fresh engine's logits."""
    from paper_2310_18859_b200 import MemoryBudget, PredictorConfig, PredictorNet, Rng, serve_sida
    from paper_2310_18859_b200.engine import SidaEngine

    model = make_model()
    pred = PredictorNet(PredictorConfig(), BASE["d_model"], BASE["num_layers"],
                        BASE["num_experts"], Rng(1))
    budget = MemoryBudget(3 * model.expert_bytes_each())
    small = make_stream(model, 4, seed=3)
    big = make_stream(model, 7, seed=4, batch_size=9, t_len=(10, 13))
    want = {name: serve_sida(model, pred, b, budget, compute_hit_rate=False).logits
            for name, b in (("small", small), ("big", big))}
    eng = SidaEngine(model, pred, budget)
    for name, b in (("small", small), ("big", big), ("small", small), ("big", big)):
        got = serve_sida(model, pred, b, budget, engine=eng, compute_hit_rate=False).logits
        assert len(got) == len(want[name])
        for a, c in zip(want[name], got):
            assert np.array_equal(a, c)
