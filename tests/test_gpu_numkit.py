"""GPU numeric API (paper_2310_18859_b200.numkit, router_scores,
moe_layer_forward) against the reference's own known answers: the golden
numkit fixture written by the reference (tests/golden/make_golden.py), the
reference test cases of ref tests/test_numkit.py and tests/test_moe.py:49-115
restated, and the oracle. Bars: sparsemax and top-k indices bit-exact;
softmax / router_scores within 4 ulp-scale relative error (1e-15 relative +
1e-300 absolute: GPU exp and a tree sum instead of numpy's); the fp64
single-token expert mixture within 1e-12 (the reference's own tolerance)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import numkit as onk

pytestmark = pytest.mark.gpu


def _api():
    import paper_2310_18859_b200 as p

    return p


def test_golden_numkit_fixture(cuda_device):
    p = _api()
    g = load_golden("numkit")
    for i in range(9):
        z = g[f"sparsemax_in_{i}"]
        np.testing.assert_array_equal(p.sparsemax(z[None])[0], g[f"sparsemax_out_{i}"])
        np.testing.assert_allclose(p.softmax(z), g[f"softmax_out_{i}"], rtol=1e-15, atol=1e-300)
        kk = g[f"topk_out_{i}"].size
        np.testing.assert_array_equal(p.topk(z, kk), g[f"topk_out_{i}"])
    np.testing.assert_array_equal(p.topk_rows(g["ties_in"], 3), g["ties_top3"])


def test_sparsemax_known_values_and_brute_force(cuda_device):
    p = _api()
    frozen = np.array([1.1, 1.0, -5.0])
    np.testing.assert_array_equal(p.sparsemax(frozen), onk.sparsemax(frozen))
    np.testing.assert_allclose(p.sparsemax(frozen), [0.55, 0.45, 0.0], atol=1e-15)
    rng = np.random.default_rng(7)
    z = rng.normal(0, 2.0, (64, 40))
    z[3, :5] = 1.25  # ties
    np.testing.assert_array_equal(p.sparsemax(z), onk.sparsemax(z))
    wide = rng.normal(0, 1.0, (3, 5000))  # > one bitonic tile; 2-D path
    np.testing.assert_array_equal(p.sparsemax(wide), onk.sparsemax(wide))
    s = p.sparsemax(z)
    np.testing.assert_allclose(s.sum(axis=1), 1.0, atol=1e-12)
    assert (s >= 0).all()


def test_softmax_rows_and_shapes(cuda_device):
    p = _api()
    rng = np.random.default_rng(8)
    z = rng.normal(0, 3.0, (5, 7, 33))
    got = p.softmax(z)
    assert got.shape == z.shape
    np.testing.assert_allclose(got, onk.softmax(z), rtol=1e-15, atol=1e-300)
    np.testing.assert_allclose(p.softmax(np.array([np.log(2.0), 0.0])), [2 / 3, 1 / 3],
                               atol=1e-15)
    np.testing.assert_allclose(p.softmax(np.array([1000.0, 0.0])), [1.0, 0.0], atol=1e-300)


def test_topk_ties_and_contracts(cuda_device):
    p = _api()
    from paper_2310_18859_b200 import ContractError

    np.testing.assert_array_equal(p.topk(np.array([1.0, 3.0, 3.0, 2.0]), 3), [1, 2, 3])
    np.testing.assert_array_equal(p.topk(np.array([0.0, -0.0, 0.0]), 3), [0, 1, 2])
    rng = np.random.default_rng(9)
    z = rng.integers(0, 4, (50, 64)).astype(np.float64)  # many ties
    np.testing.assert_array_equal(p.topk_rows(z, 10), np.argsort(-z, axis=1, kind="stable")[:, :10])
    for bad in (lambda: p.topk(np.ones((2, 2)), 1), lambda: p.topk(np.ones(3), 4),
                lambda: p.topk(np.ones(3), 0), lambda: p.softmax(np.array([np.nan])),
                lambda: p.sparsemax(np.array([])), lambda: p.topk_rows(np.ones((2, 3)), 5)):
        with pytest.raises(ContractError):
            bad()


# ref tests/test_moe.py:49-66
def test_router_scores(cuda_device):
    p = _api()
    from paper_2310_18859_b200 import ContractError

    rng = np.random.default_rng(1)
    x, w_r = rng.normal(0, 1, 6), rng.normal(0, 1, (6, 4))
    np.testing.assert_allclose(p.router_scores(x, w_r), onk.softmax(w_r.T @ x), rtol=1e-14)
    with pytest.raises(ContractError):
        p.router_scores(np.ones(3), np.zeros((4, 2)))
    with pytest.raises(ContractError):
        p.router_scores(np.array([np.inf, 0.0]), np.zeros((2, 2)))


def _experts(rng, K, d, h):
    return (rng.normal(0, 1, (K, d, h)), rng.normal(0, 1, (K, h)), rng.normal(0, 1, (K, h, d)),
            rng.normal(0, 1, (K, d)))


# ref tests/test_moe.py:67-115 (Eq. 1, single embedding)
def test_moe_layer_forward_reference_cases(cuda_device):
    p = _api()
    from paper_2310_18859_b200 import ContractError

    rng = np.random.default_rng(2)
    experts = _experts(rng, 4, 6, 5)
    x = rng.normal(0, 1, 6)
    w1, b1, w2, b2 = experts
    f3 = np.maximum(x @ w1[3] + b1[3], 0) @ w2[3] + b2[3]
    np.testing.assert_allclose(p.moe_layer_forward(x, np.array([3]), np.array([0.7]), experts),
                               0.7 * f3, atol=1e-12)
    # degenerate equal experts
    w1, b1, w2, b2 = (a.copy() for a in _experts(rng, 2, 6, 5))
    w1[1], b1[1], w2[1], b2[1] = w1[0], b1[0], w2[0], b2[0]
    f0 = np.maximum(x @ w1[0] + b1[0], 0) @ w2[0] + b2[0]
    np.testing.assert_allclose(
        p.moe_layer_forward(x, np.array([0, 1]), np.array([0.5, 0.5]), (w1, b1, w2, b2)), f0,
        atol=1e-12)
    # soft routing equals the dense oracle
    experts = _experts(rng, 5, 6, 5)
    alphas = onk.softmax(rng.normal(0, 1, 5))
    w1, b1, w2, b2 = experts
    dense = sum(alphas[i] * (np.maximum(x @ w1[i] + b1[i], 0) @ w2[i] + b2[i]) for i in range(5))
    np.testing.assert_allclose(p.moe_layer_forward(x, np.arange(5), alphas, experts), dense,
                               atol=1e-12)
    # only the selected experts are evaluated
    experts = _experts(rng, 6, 4, 3)
    counts = np.zeros(6, dtype=np.int64)
    p.moe_layer_forward(rng.normal(0, 1, 4), np.array([1, 4]), np.array([0.6, 0.4]), experts,
                        eval_counts=counts)
    assert counts.tolist() == [0, 1, 0, 0, 1, 0]
    # contract errors
    experts = _experts(rng, 3, 4, 3)
    for sel, al in (([3], [1.0]), ([], []), ([0], [-0.1]), ([-1], [1.0])):
        with pytest.raises(ContractError):
            p.moe_layer_forward(np.ones(4), np.array(sel, dtype=np.int64), np.array(al), experts)


def test_moe_layer_forward_switch_shape(cuda_device):
    """Switch-base expert width (d=768, h=3072), top-2 mixture vs numpy f64."""
    p = _api()
    rng = np.random.default_rng(3)
    d, h = 768, 3072
    experts = tuple(a * 0.03 for a in _experts(rng, 4, d, h))
    x = rng.normal(0, 1, d)
    w1, b1, w2, b2 = experts
    ref = sum(a * (np.maximum(x @ w1[e] + b1[e], 0) @ w2[e] + b2[e])
              for e, a in ((2, 0.6), (0, 0.3)))
    got = p.moe_layer_forward(x, np.array([2, 0]), np.array([0.6, 0.3]), experts)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
