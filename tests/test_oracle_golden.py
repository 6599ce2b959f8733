"""Pin the CPU oracle to the real reference's outputs (tests/golden/).

The fixtures were produced by tests/golden/make_golden.py running the
reference package itself; these tests run on CPU only.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import moe as omoe
from oracle import numkit as onk
from oracle import offload as ooff
from oracle import permute as operm
from oracle import predictor as opred


def _digest(params):
    h = hashlib.sha256()
    for name in params:
        h.update(name.encode())
        h.update(np.ascontiguousarray(params[name], dtype=np.float64).tobytes())
    return h.hexdigest()


class TestNumkit:
    g = load_golden("numkit")

    @pytest.mark.parametrize("i", range(9))
    def test_sparsemax_softmax_topk(self, i):
        z = self.g[f"sparsemax_in_{i}"]
        np.testing.assert_allclose(onk.sparsemax(z[None])[0], self.g[f"sparsemax_out_{i}"],
                                   rtol=0, atol=1e-15)
        np.testing.assert_allclose(onk.softmax(z), self.g[f"softmax_out_{i}"], rtol=1e-15)
        kk = min(3, z.size)
        np.testing.assert_array_equal(onk.topk_rows(z, kk), self.g[f"topk_out_{i}"])

    def test_frozen_sparsemax_value(self):
        # ref tests/test_numkit.py:86-90
        np.testing.assert_allclose(onk.sparsemax(np.array([[1.1, 1.0, -5.0]]))[0],
                                   [0.55, 0.45, 0.0], atol=1e-15)

    def test_topk_ties_to_lower_index(self):
        np.testing.assert_array_equal(onk.topk_rows(self.g["ties_in"], 3), self.g["ties_top3"])

    def test_sigmoid(self):
        np.testing.assert_allclose(onk.sigmoid(self.g["sigmoid_in"]), self.g["sigmoid_out"],
                                   rtol=1e-15)

    def test_bf16_rounding_is_rne(self):
        x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5e-3, 3.0e38])
        bits = onk.bf16_bits(x)
        back = onk.bf16_to_f64(bits)
        assert back[0] == 1.0 and back[1] == 1.0  # tie to even
        assert back[2] == 1.0 + 2 ** -7
        import torch

        t = torch.tensor(x, dtype=torch.float32).to(torch.bfloat16)
        np.testing.assert_array_equal(t.view(torch.int16).numpy().view(np.uint16), bits)


def _shapes(name):
    meta = json.load(open(os.path.join(GOLDEN, name + ".json")))
    c = meta["config"]
    shape = omoe.MoEShape(**c)
    pshape = opred.PredictorShape(c["d_model"], c["num_layers"], c["num_experts"],
                                  **meta["predictor"])
    return meta, shape, pshape


@pytest.mark.parametrize("name", ["tiny", "c0"])
class TestModelFixtures:
    def test_init_matches_reference_rng(self, name):
        meta, shape, pshape = _shapes(name)
        assert _digest(omoe.init_params(shape, 0)) == meta["moe_digest"]
        assert _digest(opred.init_params(pshape, 1)) == meta["predictor_digest"]

    def test_hash_table_forward_and_permutation(self, name):
        meta, shape, pshape = _shapes(name)
        g = load_golden(name)
        params = omoe.bf16_params(omoe.init_params(shape, 0))
        pparams = opred.init_params(pshape, 1)
        lengths = g["lengths"].tolist()
        toks = g["tokens"]
        seqs = np.split(toks, np.cumsum(lengths)[:-1])
        emb = lambda t: omoe.embed(params, shape, t)  # noqa: E731
        np.testing.assert_allclose(opred.forward(pparams, emb(seqs[0])), g["pred_logits_seq0"],
                                   rtol=1e-12, atol=1e-13)
        for k in meta["ks"]:
            ids, alphas = opred.build_hash_table(pparams, seqs, k, emb)
            np.testing.assert_array_equal(ids, g[f"ids_k{k}"])
            np.testing.assert_allclose(alphas, g[f"alphas_k{k}"], rtol=1e-12)
            for layer in range(shape.num_layers):
                hist, off, perm, inv = operm.permute_layer(ids[layer], shape.num_experts)
                np.testing.assert_array_equal(perm, g[f"perm_k{k}_l{layer}"])
                np.testing.assert_array_equal(hist, g[f"hist_k{k}_l{layer}"])
                assert off[-1] == ids[layer].size
                np.testing.assert_array_equal(perm[inv], np.arange(perm.size))
            x = g[f"layer0_in_k{k}"]
            t0 = lengths[0]
            np.testing.assert_allclose(
                omoe.moe_apply(params, 0, x, ids[0, :t0], alphas[0, :t0]),
                g[f"layer0_out_k{k}"], rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(
                omoe.moe_apply_grouped(params, 0, x, ids[0, :t0], alphas[0, :t0]),
                g[f"layer0_out_k{k}"], rtol=1e-11, atol=1e-12)
            if name == "tiny" or k == 1:
                logits = omoe.forward_external(params, shape, seqs, ids, alphas)
                np.testing.assert_allclose(logits, g[f"logits_k{k}"], rtol=1e-10, atol=1e-12)


def test_planner_replays_reference_plans():
    cases = json.load(open(os.path.join(GOLDEN, "planner.json")))
    for case in cases:
        eb = case["expert_bytes"]
        budget = case["slots"] * eb
        resident, fifo, used = {}, [], 0
        for b in case["batches"]:
            req = [set(r) for r in b["required"]]
            groups = ooff.plan(req, resident, fifo, used, budget, eb,
                               case["bandwidth"], case["latency"])
            assert len(groups) == len(b["groups"])
            for mine, ref in zip(groups, b["groups"]):
                assert [[op, list(k)] for op, k in mine["steps"]] == ref["steps"]
                assert mine["prefetchable"] == ref["prefetchable"]
                assert mine["transfer_s"] == pytest.approx(ref["transfer_s"], rel=1e-12)
            for gr in groups:
                used = ooff.apply_group(resident, fifo, used, gr, budget, eb)
            assert [list(k) for k in fifo] == b["fifo_after"]


ROUTER_CFGS = {
    "tiny": dict(vocab_size=64, d_model=32, num_layers=2, num_experts=8, expert_hidden=64,
                 max_seq_len=16, routing_k=1, num_classes=3),
    "tiny_r2": dict(vocab_size=64, d_model=32, num_layers=3, num_experts=6, expert_hidden=64,
                    max_seq_len=16, routing_k=2, num_classes=3),
    "c0": dict(vocab_size=512, d_model=256, num_layers=2, num_experts=8, expert_hidden=1024,
               max_seq_len=128, routing_k=1, num_classes=4),
}


@pytest.mark.parametrize("name", sorted(ROUTER_CFGS))
def test_router_mode_matches_reference(name):
    """Router-mode forward, OracleHasher table and hash_hit_rate
    (ref moe.py:296-306, predictor.py:413-449) against the reference's outputs."""
    shape = omoe.MoEShape(**ROUTER_CFGS[name])
    g = load_golden("router_" + name)
    params = omoe.bf16_params(omoe.init_params(shape, 0))
    pparams = opred.init_params(opred.PredictorShape(shape.d_model, shape.num_layers,
                                                     shape.num_experts), 1)
    seqs = np.split(g["tokens"], np.cumsum(g["lengths"])[:-1])
    logits, sel, al, probs = omoe.forward_router(params, shape, seqs)
    np.testing.assert_array_equal(sel, g["selected"])
    np.testing.assert_allclose(al, g["alphas"], rtol=1e-12)
    np.testing.assert_allclose(probs, g["probs"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(logits, g["logits"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(logits, g["standard_logits_b0"], rtol=1e-10, atol=1e-12)
    emb = lambda t: omoe.embed(params, shape, t)  # noqa: E731
    for key in g.files:
        if key.startswith("oracle_ids_k"):
            k = int(key[len("oracle_ids_k"):])
            ids, alphas = opred.oracle_table(probs, k)
            np.testing.assert_array_equal(ids, g[key])
            np.testing.assert_allclose(alphas, g[f"oracle_alphas_k{k}"], rtol=1e-12)
            pids, _ = opred.build_hash_table(pparams, seqs, k, emb)
            np.testing.assert_array_equal(pids, g[f"pred_ids_k{k}"])
            assert opred.hash_hit_rate([pids], [sel], k) == float(g[f"hit_rate_k{k}"])
    assert float(g["oracle_serve_hit_rate"]) == 1.0


def test_ensure_layer_resident_replays_reference():
    cases = json.load(open(os.path.join(GOLDEN, "ensure.json")))
    for case in cases:
        eb = case["expert_bytes"]
        resident, fifo, used = {}, [], 0
        for call in case["calls"]:
            steps, used = ooff.ensure_layer(resident, fifo, used, call["layer"], call["required"],
                                            case["slots"] * eb, eb)
            assert [[op, list(k)] for op, k in steps] == call["steps"]
            assert [list(k) for k in fifo] == call["fifo_after"]
