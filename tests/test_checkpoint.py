"""Checkpoint containers (ref checkpoint.py:1-86, moe.py:581-596,
predictor.py:550-571) against files written by the reference itself
(tests/golden/mini64.sidamoe / .sidahsh, made by make_golden.py --checkpoint).
Host-only: the container code needs no GPU."""

import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import moe as omoe
from oracle import predictor as opred

MOE = os.path.join(GOLDEN, "mini64.sidamoe")
HSH = os.path.join(GOLDEN, "mini64.sidahsh")
SHAPE = omoe.MoEShape(vocab_size=64, d_model=64, num_layers=2, num_experts=4, expert_hidden=128,
                      max_seq_len=16, routing_k=1, num_classes=3)


def test_reference_moe_container_reads_back_the_reference_draws():
    from paper_2310_18859_b200.checkpoint import MOE_MAGIC, load_container, map_container

    cfg, tensors = load_container(MOE, MOE_MAGIC)
    assert cfg == SHAPE.__dict__
    ref = omoe.init_params(SHAPE, 0)  # the reference's Rng(0) draws, bit-for-bit
    assert list(tensors) == list(ref)  # declared order
    for k, v in ref.items():
        np.testing.assert_array_equal(tensors[k], v)
    _, views = map_container(MOE, MOE_MAGIC)
    assert all(not v.flags.writeable for v in views.values())


def test_container_write_is_byte_identical_to_the_reference(tmp_path):
    from paper_2310_18859_b200.checkpoint import (MOE_MAGIC, PREDICTOR_MAGIC, load_container,
                                                  save_container)

    for path, magic in ((MOE, MOE_MAGIC), (HSH, PREDICTOR_MAGIC)):
        cfg, tensors = load_container(path, magic)
        out = tmp_path / "copy.bin"
        save_container(out, magic, cfg, tensors)
        assert out.read_bytes() == open(path, "rb").read()


def test_reference_predictor_container():
    from paper_2310_18859_b200.checkpoint import PREDICTOR_MAGIC, load_container

    cfg, tensors = load_container(HSH, PREDICTOR_MAGIC)
    assert (cfg["d_model"], cfg["num_moe_layers"], cfg["num_experts"]) == (64, 2, 4)
    ref = opred.init_params(opred.PredictorShape(64, 2, 4, compress_dim=8, lstm_hidden=16), 1)
    for k, v in ref.items():
        np.testing.assert_array_equal(tensors[k], v)


def test_load_predictor_round_trip(tmp_path):
    from paper_2310_18859_b200.checkpoint import load_predictor, save_predictor

    net = load_predictor(HSH)
    assert net.config.compress_dim == 8 and net.config.lstm_hidden == 16
    out = tmp_path / "p.sidahsh"
    save_predictor(net, out)
    assert out.read_bytes() == open(HSH, "rb").read()


@pytest.mark.parametrize("damage", ["magic", "truncate", "trailing", "names"])
def test_container_contract_errors(tmp_path, damage):
    from paper_2310_18859_b200.checkpoint import (MOE_MAGIC, PREDICTOR_MAGIC, load_container,
                                                  load_predictor, save_container)
    from paper_2310_18859_b200.errors import ContractError

    bad = tmp_path / "bad.bin"
    shutil.copy(HSH, bad)
    raw = bad.read_bytes()
    if damage == "magic":
        with pytest.raises(ContractError, match="bad magic"):
            load_container(bad, MOE_MAGIC)
        return
    if damage == "truncate":
        bad.write_bytes(raw[:-9])
        with pytest.raises(ContractError, match="truncated"):
            load_container(bad, PREDICTOR_MAGIC)
    elif damage == "trailing":
        bad.write_bytes(raw + b"\0")
        with pytest.raises(ContractError, match="trailing"):
            load_container(bad, PREDICTOR_MAGIC)
    else:
        cfg, tensors = load_container(HSH, PREDICTOR_MAGIC)
        tensors["extra"] = np.zeros(3)
        save_container(bad, PREDICTOR_MAGIC, cfg, tensors)
        with pytest.raises(ContractError, match="names"):
            load_predictor(bad)
