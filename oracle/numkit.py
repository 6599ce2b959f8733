"""Arithmetic contract of the hot path (oracle; test infrastructure only).

Restates ref `pkg/src/sida/numkit.py` for the forward ops the kernels must
reproduce, plus the bf16 rounding both sides share.
"""

from __future__ import annotations

import numpy as np


def make_rng(seed: int) -> np.random.Generator:
    """PCG64 over SeedSequence(seed) -- the stream ref `numkit.py:172-185`
    (`Rng.__init__`) draws from, so parameter inits are bit-identical."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(int(seed))))


def softmax(z: np.ndarray) -> np.ndarray:
    """Max-shifted softmax over the last axis (ref `numkit.py:28-33`)."""
    z = np.asarray(z, dtype=np.float64)
    m = z.max(axis=-1, keepdims=True)
    ez = np.exp(z - m)
    return ez / ez.sum(axis=-1, keepdims=True)


def sparsemax(z: np.ndarray) -> np.ndarray:
    """Simplex projection per row (ref `numkit.py:42-60`).

    Sorted-descending closed form: k_z = #{k : 1 + k*z_(k) > S_k} with S the
    running sum of the sorted row, tau = (S_{k_z} - 1)/k_z, out = max(z-tau,0).
    """
    z = np.asarray(z, dtype=np.float64)
    shape = z.shape
    rows = z.reshape(-1, shape[-1])
    desc = np.sort(rows, axis=1)[:, ::-1]
    run = np.cumsum(desc, axis=1)
    k = np.arange(1, rows.shape[1] + 1, dtype=np.float64)
    kz = np.sum(1.0 + k * desc > run, axis=1)
    tau = (run[np.arange(rows.shape[0]), kz - 1] - 1.0) / kz
    return np.maximum(rows - tau[:, None], 0.0).reshape(shape)


def topk_rows(z: np.ndarray, k: int) -> np.ndarray:
    """Descending order, ties to the lower index (ref `numkit.py:87-93`)."""
    return np.argsort(-np.asarray(z), axis=-1, kind="stable")[..., :k]


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Split-branch stable logistic (ref `numkit.py:104-110`)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    nonneg = x >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-x[nonneg]))
    ex = np.exp(x[~nonneg])
    out[~nonneg] = ex / (1.0 + ex)
    return out


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float64 -> float32 (RNE) -> bfloat16 (RNE), returned as uint16 bits.

    The single rounding recipe shared by the oracle and the GPU weight
    upload, so both sides hold bit-identical bf16 parameters (SURVEY §8(c)
    parity protocol)."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Values of ``x`` after bf16 rounding, as float64."""
    return bf16_to_f64(bf16_bits(x))
