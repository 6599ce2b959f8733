"""load_moe / save_moe on the GPU model: a reference-written checkpoint
(tests/golden/mini64.sidamoe) streamed into pinned bf16 expert slabs serves
the same logits as the oracle on the bf16 weights, and save_moe writes back
exactly the bf16 values (byte-identical to the container of the rounded
parameters)."""

import numpy as np
import pytest

from oracle import moe as omoe
from oracle import numkit as onk
from oracle import predictor as opred
from test_checkpoint import HSH, MOE, SHAPE
from test_gpu_kernels import close_rms

pytestmark = pytest.mark.gpu


def test_load_moe_serves_reference_checkpoint(cuda_device):
    from paper_2310_18859_b200 import MemoryBudget, SequenceBatch, serve_sida
    from paper_2310_18859_b200.checkpoint import load_moe, load_predictor
    from paper_2310_18859_b200.predictor import build_hash_table

    model = load_moe(MOE)
    net = load_predictor(HSH)
    params = omoe.bf16_params(omoe.init_params(SHAPE, 0))
    pparams = opred.init_params(opred.PredictorShape(64, 2, 4, compress_dim=8, lstm_hidden=16), 1)
    g = np.random.default_rng(4)
    seqs = [g.integers(0, 64, size=n) for n in (16, 7, 12, 16)]
    batch = SequenceBatch(0, seqs)
    table = build_hash_table(net, batch, 1, model.embed)
    emb = lambda t: params["tok_emb"][t] + params["pos_emb"][: len(t)]  # noqa: E731
    ids, alphas = opred.build_hash_table(pparams, seqs, 1, emb)
    np.testing.assert_array_equal(table.ids, ids)
    rep = serve_sida(model, net, [batch], MemoryBudget(3 * model.expert_bytes_each()),
                     compute_hit_rate=False)
    ref = omoe.forward_external(params, SHAPE, seqs, ids, alphas)
    close_rms(rep.logits[0], ref, 2e-2)


def test_save_moe_round_trip(cuda_device, tmp_path):
    from paper_2310_18859_b200.checkpoint import (MOE_MAGIC, load_container, load_moe, save_container,
                                                  save_moe)

    model = load_moe(MOE)
    out = tmp_path / "b200.sidamoe"
    save_moe(model, out)
    cfg, tensors = load_container(MOE, MOE_MAGIC)
    want = tmp_path / "rounded.sidamoe"
    save_container(want, MOE_MAGIC, cfg, {k: onk.round_bf16(v) for k, v in tensors.items()})
    assert out.read_bytes() == want.read_bytes()
    again = tmp_path / "again.sidamoe"
    save_moe(load_moe(out), again)
    assert again.read_bytes() == out.read_bytes()
