"""Router mode on the GPU (the teacher path): the fused softmax + top-k router
kernel, router-mode model_forward, OracleHasher, hash hit rate and
serve_standard, against the reference's fixtures (tests/golden/router_*.npz,
made by running the reference) and the oracle (ref moe.py:296-306,
predictor.py:413-449, pipeline.py:326-429)."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import moe as omoe
from oracle import numkit as onk
from test_gpu_kernels import close_rms

pytestmark = pytest.mark.gpu

CFGS = {
    "tiny": dict(vocab_size=64, d_model=32, num_layers=2, num_experts=8, expert_hidden=64,
                 max_seq_len=16, routing_k=1, num_classes=3),
    "tiny_r2": dict(vocab_size=64, d_model=32, num_layers=3, num_experts=6, expert_hidden=64,
                    max_seq_len=16, routing_k=2, num_classes=3),
    "c0": dict(vocab_size=512, d_model=256, num_layers=2, num_experts=8, expert_hidden=1024,
               max_seq_len=128, routing_k=1, num_classes=4),
}


def _router_gpu(x32: np.ndarray, w32: np.ndarray, k: int):
    from paper_2310_18859_b200 import _lib

    dev = torch.device("cuda")
    n, d = x32.shape
    K = w32.shape[1]
    x = torch.from_numpy(np.ascontiguousarray(x32)).to(dev)
    w = torch.from_numpy(np.ascontiguousarray(w32)).to(dev)
    ids = torch.empty((n, k), dtype=torch.int32, device=dev)
    al = torch.empty((n, k), dtype=torch.float64, device=dev)
    al32 = torch.empty((n, k), dtype=torch.float32, device=dev)
    pr = torch.empty((n, K), dtype=torch.float32, device=dev)
    _lib.check(_lib.lib().sida_router_topk(x.data_ptr(), n, d, w.data_ptr(), K, k, pr.data_ptr(),
                                           ids.data_ptr(), al.data_ptr(), al32.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return ids.cpu().numpy(), al.cpu().numpy(), pr.cpu().numpy()


def _check_router(x32, w32, k):
    """GPU selection vs the oracle's softmax/topk_rows on the same fp32
    inputs: probabilities within 2e-6, ids identical except where the k-th
    and (k+1)-th probabilities are closer than the fp32 logit error."""
    ids, al, pr = _router_gpu(x32, w32, k)
    probs = onk.softmax(x32.astype(np.float64) @ w32.astype(np.float64))
    ref = onk.topk_rows(probs, k)
    np.testing.assert_allclose(pr, probs, rtol=0, atol=2e-6)
    np.testing.assert_allclose(al, np.take_along_axis(pr.astype(np.float64), ids, 1), rtol=1e-6)
    srt = -np.sort(-probs, axis=1)
    gap = np.min(np.abs(np.diff(srt[:, : min(k + 1, probs.shape[1])], axis=1)), axis=1) \
        if probs.shape[1] > 1 else np.ones(len(probs))
    clear = gap > 1e-5
    np.testing.assert_array_equal(ids[clear], ref[clear])
    # every row, near ties included: the picked experts carry the top-k
    # probabilities in descending order (a wrong pick would show as a gap)
    np.testing.assert_allclose(np.take_along_axis(probs, ids, 1), srt[:, :k], rtol=0, atol=4e-6)
    return ids, al, pr


@pytest.mark.parametrize("name", sorted(CFGS))
def test_router_kernel_on_reference_activations(cuda_device, name):
    shape = omoe.MoEShape(**CFGS[name])
    g = load_golden("router_" + name)
    params = omoe.bf16_params(omoe.init_params(shape, 0))
    x32 = g["router_in_l0"].astype(np.float32)
    w32 = params["block0.w_r"].astype(np.float32)
    for k in sorted({1, shape.routing_k, shape.num_experts}):
        _check_router(x32, w32, k)
    # the reference's own layer-0 selections on its float64 activations
    ids, _, _ = _router_gpu(x32, w32, shape.routing_k)
    agree = np.mean(ids == g["selected"][0])
    assert agree > 0.99, agree


@pytest.mark.parametrize("n,d,K,k", [(1, 1, 1, 1), (5, 7, 3, 2), (1000, 768, 128, 2),
                                     (4099, 768, 256, 4), (300, 64, 64, 64), (33, 100, 17, 5)])
def test_router_kernel_shapes(cuda_device, n, d, K, k):
    g = np.random.default_rng(n + d + K)
    x32 = g.normal(0, 1, (n, d)).astype(np.float32)
    w32 = onk.round_bf16(g.normal(0, 1 / np.sqrt(d), (d, K))).astype(np.float32)
    _check_router(x32, w32, k)


def test_router_ties_go_to_the_lower_index(cuda_device):
    g = np.random.default_rng(5)
    w = onk.round_bf16(g.normal(0, 0.1, (64, 12))).astype(np.float32)
    w[:, 9] = w[:, 3]   # experts 3 and 9 always tie
    w[:, 11] = w[:, 0]  # experts 0 and 11 always tie
    x = g.normal(0, 1, (500, 64)).astype(np.float32)
    ids, al, pr = _router_gpu(x, w, 12)
    pos = {e: np.argmax(ids == e, axis=1) for e in (0, 3, 9, 11)}
    assert np.all(pos[3] < pos[9]) and np.all(pos[0] < pos[11])
    np.testing.assert_array_equal(pr[:, 3], pr[:, 9])


def test_router_contracts(cuda_device):
    from paper_2310_18859_b200.errors import ContractError, NativeLibraryError

    x = np.zeros((4, 8), np.float32)
    with pytest.raises(ContractError):
        _router_gpu(x, np.zeros((8, 4), np.float32), 5)
    with pytest.raises(NativeLibraryError):
        _router_gpu(x, np.zeros((8, 300), np.float32), 1)


# ----------------------------------------------------------------- full router-mode paths
def _c0():
    from paper_2310_18859_b200 import MoEConfig, MoEModel, SequenceBatch

    shape = omoe.MoEShape(**CFGS["c0"])
    params = omoe.bf16_params(omoe.init_params(shape, 0))
    model = MoEModel(MoEConfig(**CFGS["c0"]), params=params)
    g = load_golden("router_c0")
    seqs = np.split(g["tokens"], np.cumsum(g["lengths"])[:-1])
    return model, SequenceBatch(0, list(seqs)), g, seqs


def _clear_top1(probs):
    s = -np.sort(-probs, axis=-1)
    return (s[..., 0] - s[..., 1]) > 1e-2


def test_model_forward_router_c0_vs_reference(cuda_device):
    from paper_2310_18859_b200 import model_forward

    model, batch, g, _ = _c0()
    logits, trace = model_forward(model, batch, mode="router")
    clear = _clear_top1(g["probs"])
    np.testing.assert_array_equal(trace.selected[..., 0][clear], g["selected"][..., 0][clear])
    assert np.mean(trace.selected == g["selected"]) > 0.98
    np.testing.assert_allclose(trace.probs, g["probs"], rtol=0, atol=5e-2)
    assert trace.probs.shape == g["probs"].shape and trace.alphas.shape == g["alphas"].shape
    if np.array_equal(trace.selected, g["selected"]):
        close_rms(logits, g["logits"], 2e-2)
    # unconditionally: the oracle forward driven by the GPU's own selections
    shape = omoe.MoEShape(**CFGS["c0"])
    params = omoe.bf16_params(omoe.init_params(shape, 0))
    seqs = np.split(g["tokens"], np.cumsum(g["lengths"])[:-1])
    ref = omoe.forward_external(params, shape, seqs, trace.selected, trace.alphas)
    close_rms(logits, ref, 2e-2)


def test_oracle_hasher_and_hit_rate_c0(cuda_device):
    from paper_2310_18859_b200 import (MemoryBudget, OracleHasher, PredictorConfig, PredictorNet,
                                       hash_hit_rate, model_forward, serve_sida)
    from oracle import predictor as opred

    model, batch, g, seqs = _c0()
    table = OracleHasher(model).build_table(batch, 1)
    _, trace = model_forward(model, batch, mode="router")
    np.testing.assert_array_equal(table.ids, trace.selected)
    np.testing.assert_allclose(table.alphas, trace.alphas, rtol=1e-12)
    assert hash_hit_rate([table], [trace], 1) == 1.0
    eb = model.expert_bytes_each()
    rep = serve_sida(model, None, [batch], MemoryBudget(16 * eb), eval_top_k=1)
    assert rep.mode == "oracle" and rep.hit_rate == 1.0
    # predictor hasher: hit rate against the GPU teacher = the reference's
    # value up to tokens whose teacher top-1 is a near tie
    net = PredictorNet(PredictorConfig(), 256, 2, 8,
                       params=opred.init_params(opred.PredictorShape(256, 2, 8), 1))
    rep = serve_sida(model, net, [batch], MemoryBudget(16 * eb), eval_top_k=1)
    assert rep.mode == "sida"
    n = g["selected"][..., 0].size
    slack = np.sum(~_clear_top1(g["probs"])) / n
    assert abs(rep.hit_rate - float(g["hit_rate_k1"])) <= slack + 1e-12


def test_serve_standard_c0(cuda_device):
    from paper_2310_18859_b200 import MemoryBudget, SequenceBatch, model_forward, serve_standard
    from paper_2310_18859_b200.errors import ContractError, UnservableError

    model, batch, g, seqs = _c0()
    eb = model.expert_bytes_each()
    b1 = SequenceBatch(1, list(seqs[::-1]))
    ref0, _ = model_forward(model, batch, mode="router")
    ref1, _ = model_forward(model, b1, mode="router")
    for slots in (4, 1, 16):
        rep = serve_standard(model, [batch, b1], MemoryBudget(slots * eb))
        assert rep.mode == "standard" and rep.eval_top_k is None
        assert rep.peak_fast_tier_bytes <= slots * eb
        np.testing.assert_array_equal(rep.logits[0], ref0)  # budgets only move time
        np.testing.assert_array_equal(rep.logits[1], ref1)
        assert rep.expert_loads > 0
        assert all(r["selection_s"] >= 0 for r in rep.batch_records)
        if slots == 4:  # the reference's run used the same 4-slot budget
            assert rep.peak_fast_tier_bytes // eb == int(g["standard_peak"])
    with pytest.raises(UnservableError):
        serve_standard(model, [batch], MemoryBudget(eb - 1))
    with pytest.raises(ContractError):
        serve_standard(model, [], MemoryBudget(eb))
