"""End-to-end GPU serving parity: the external-table forward and serve_sida
against the reference fixtures and against themselves under budgets
(ref tests/test_pipeline.py:127-166 contracts)."""

import numpy as np
import pytest
import torch

from test_gpu_kernels import _hash_fixture, close_rms

pytestmark = pytest.mark.gpu


def test_model_forward_c0_logits_vs_reference(cuda_device):
    from paper_2310_18859_b200.moe import model_forward
    from paper_2310_18859_b200.predictor import build_hash_table

    meta, model, net, batch, g, params, shape = _hash_fixture("c0")
    table = build_hash_table(net, batch, 1, model.embed)
    logits, trace = model_forward(model, batch, mode="external", table=table)
    close_rms(logits, g["logits_k1"], 2e-2)
    np.testing.assert_array_equal(trace.selected, g["ids_k1"])


def test_model_forward_layer_isolation_c0(cuda_device):
    """Per-layer isolation: feed the oracle moe_apply the GPU's
    own attention output for each layer."""
    from oracle import moe as omoe
    from paper_2310_18859_b200.moe import BatchLayout
    from paper_2310_18859_b200.offload import ExpertStore
    from paper_2310_18859_b200.predictor import build_hash_table

    meta, model, net, batch, g, params, shape = _hash_fixture("c0")
    table = build_hash_table(net, batch, 1, model.embed)
    dt = table.on_device(model)
    torch.cuda.current_stream().wait_event(dt.ready)
    lay = BatchLayout(batch.lengths, dt.tokens_for(model, batch), model.device)
    x = model.embed_layout(lay)
    store = ExpertStore.full(model)
    ids, al = table.ids, table.alphas
    for layer in range(shape.num_layers):
        xa = model.attention_mix(layer, x, lay)
        x = store.run_layer(model, layer, xa, dt)
        xin = xa.cpu().numpy().astype(np.float64)
        ref = omoe.moe_apply_grouped(params, layer, xin, ids[layer], al[layer])
        close_rms(x.cpu().numpy(), ref, 2e-2)


def _stream(model, n_batches, bs, t_lo, t_hi, seed=0):
    from paper_2310_18859_b200.moe import SequenceBatch

    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_batches):
        seqs = [rng.integers(0, model.config.vocab_size, size=int(rng.integers(t_lo, t_hi + 1)))
                for _ in range(bs)]
        out.append(SequenceBatch(i, seqs, [int(rng.integers(0, model.config.num_classes))
                                           for _ in seqs]))
    return out


def test_serve_sida_budget_invariance_and_determinism(cuda_device):
    from paper_2310_18859_b200.moe import model_forward
    from paper_2310_18859_b200.offload import MemoryBudget
    from paper_2310_18859_b200.pipeline import serve_sida
    from paper_2310_18859_b200.predictor import build_hash_table

    meta, model, net, batch, g, params, shape = _hash_fixture("c0")
    batches = _stream(model, 4, 3, 5, 128)
    eb = model.expert_bytes_each()
    total = model.total_expert_bytes()
    runs = []
    for slots in (16, 7, 3, 1, 16, 16, 16, 16):
        rep = serve_sida(model, net, batches, MemoryBudget(slots * eb), eval_top_k=1,
                         compute_hit_rate=False)
        assert rep.peak_fast_tier_bytes <= slots * eb
        runs.append(rep)
    base = runs[0].logits
    for rep in runs[1:]:
        for a, b in zip(base, rep.logits):
            np.testing.assert_array_equal(a, b)  # budgets only move time around
    for i, b in enumerate(batches):
        table = build_hash_table(net, b, 1, model.embed)
        lg, _ = model_forward(model, b, mode="external", table=table)
        np.testing.assert_array_equal(lg, base[i].astype(np.float32).astype(np.float64))
    assert runs[0].total_tokens == sum(b.num_tokens for b in batches)
    assert runs[3].expert_loads > runs[0].expert_loads  # 1 slot forces reloads


def test_serve_sida_k2_and_report(cuda_device, tmp_path):
    from paper_2310_18859_b200.offload import MemoryBudget
    from paper_2310_18859_b200.pipeline import serve_sida

    meta, model, net, batch, g, params, shape = _hash_fixture("tiny")
    # tiny has d=32 (not a tcgen05 shape): the bf16 FFN must refuse loudly
    from paper_2310_18859_b200.errors import NativeLibraryError

    with pytest.raises(NativeLibraryError):
        serve_sida(model, net, _stream(model, 1, 2, 3, 8), MemoryBudget(model.total_expert_bytes()))


def test_serve_sida_contracts(cuda_device):
    from paper_2310_18859_b200.errors import ContractError, UnservableError
    from paper_2310_18859_b200.offload import MemoryBudget
    from paper_2310_18859_b200.pipeline import serve_sida

    meta, model, net, batch, g, params, shape = _hash_fixture("c0")
    eb = model.expert_bytes_each()
    with pytest.raises(UnservableError):
        serve_sida(model, net, _stream(model, 1, 1, 4, 8), MemoryBudget(eb - 1))
    with pytest.raises(ContractError):
        serve_sida(model, net, [], MemoryBudget(eb))
    bad = _stream(model, 2, 1, 4, 8)
    bad[1].batch_id = 0
    with pytest.raises(ContractError):
        serve_sida(model, net, bad, MemoryBudget(eb))
    with pytest.raises(ContractError):
        serve_sida(model, net, _stream(model, 1, 1, 4, 8), MemoryBudget(eb), prefetch="never")


def test_spread_victim_policy_serves_identical_logits(cuda_device):
    """The opt-in spread victim order only changes which slots are reused and
    when copies run: logits bit-identical to the all-resident reference plan
    at every budget, with no more expert loads than the FIFO plan."""
    from paper_2310_18859_b200.engine import SidaEngine
    from paper_2310_18859_b200.offload import MemoryBudget
    from paper_2310_18859_b200.pipeline import serve_sida

    meta, model, net, batch, g, params, shape = _hash_fixture("c0")
    batches = _stream(model, 6, 3, 5, 128)
    eb = model.expert_bytes_each()
    base = serve_sida(model, net, batches, MemoryBudget(16 * eb), eval_top_k=1,
                      compute_hit_rate=False)
    for slots in (13, 7, 3, 1):
        reps = {}
        for policy in ("fifo", "spread"):
            eng = SidaEngine(model, net, MemoryBudget(slots * eb), victim_policy=policy)
            reps[policy] = serve_sida(model, net, batches, MemoryBudget(slots * eb),
                                      eval_top_k=1, compute_hit_rate=False, engine=eng)
            assert reps[policy].peak_fast_tier_bytes <= slots * eb
            for a, b in zip(base.logits, reps[policy].logits):
                np.testing.assert_array_equal(a, b)
        assert reps["spread"].expert_loads <= reps["fifo"].expert_loads
