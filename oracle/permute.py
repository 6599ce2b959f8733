"""Token permutation + histogram contract, SURVEY §8(a) row A13 (oracle).

The reference has no explicit permute: `moe_apply` gathers expert weights
per token (ref `moe.py:253-256`). The GPU path instead groups the (token,
rank) rows of one layer by expert. This restatement *is* the contract:

  flat   = ids[l].reshape(-1)           row index = global_token * k + rank
                                        (layout of ref `moe.py:14-16`)
  hist   = bincount(flat, minlength=K)
  off    = exclusive prefix sum of hist, length K + 1
  perm   = stable argsort(flat)         within an expert: ascending row
  inv    = argsort(perm)                inv[perm[p]] = p

The expert order equals `np.unique` / `sorted` in ref `predictor.py:96-100`
and `offload.py:164`, which is why the planner and the permutation agree.
"""

from __future__ import annotations

import numpy as np


def permute_layer(ids_layer: np.ndarray, num_experts: int):
    """ids_layer (N, k) -> (hist (K,), off (K+1,), perm (N*k,), inv (N*k,)), int64."""
    flat = np.asarray(ids_layer, dtype=np.int64).reshape(-1)
    if flat.size and (flat.min() < 0 or flat.max() >= num_experts):
        raise ValueError("expert index out of range")
    hist = np.bincount(flat, minlength=num_experts).astype(np.int64)
    off = np.zeros(num_experts + 1, dtype=np.int64)
    np.cumsum(hist, out=off[1:])
    perm = np.argsort(flat, kind="stable").astype(np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size, dtype=np.int64)
    return hist, off, perm, inv


def permute_all(ids: np.ndarray, num_experts: int):
    """Apply :func:`permute_layer` to every layer of an (L, N, k) table."""
    parts = [permute_layer(ids[l], num_experts) for l in range(ids.shape[0])]
    return tuple(np.stack([p[i] for p in parts]) for i in range(4))


def gather_rows(x: np.ndarray, perm: np.ndarray, k: int) -> np.ndarray:
    """x_perm[p] = x[perm[p] // k] (the optional row gather of A13)."""
    return x[np.asarray(perm) // k]
