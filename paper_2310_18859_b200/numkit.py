"""The reference's numeric API on the GPU (ref pkg/src/sida/numkit.py:19-93).

Same names, shapes, validation and exception types as the reference
(`check_finite`, `softmax`, `sparsemax`, `topk`, `topk_rows`); the arithmetic
runs in the fp64 row kernels of csrc/numkit.cu (`sida_softmax_rows_f64`,
`sida_sparsemax_rows_f64`, `sida_topk_rows_f64`). Inputs are numpy arrays
(or anything ``np.asarray`` accepts) and results come back as numpy, like
the reference. sparsemax and the top-k indices are bit-identical to the
reference; softmax agrees to a few ulp (GPU exp, tree sum). The batched
serving path never calls these: the hash kernels fuse the same arithmetic.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ContractError


def check_finite(x, name: str = "input") -> np.ndarray:
    """ref numkit.py:19-25."""
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise ContractError(f"{name} is empty")
    if not np.all(np.isfinite(x)):
        raise ContractError(f"{name} contains NaN or Inf")
    return x


def _rows(z: np.ndarray) -> tuple[torch.Tensor, tuple]:
    shape = z.shape
    flat = np.ascontiguousarray(z.reshape(-1, shape[-1]))
    return torch.from_numpy(flat).to(torch.device("cuda", torch.cuda.current_device())), shape


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def softmax(z) -> np.ndarray:
    """Stable softmax over the last axis (ref numkit.py:28-33)."""
    z = check_finite(z, "softmax input")
    d, shape = _rows(z)
    out = torch.empty_like(d)
    _lib.check(_lib.lib().sida_softmax_rows_f64(d.data_ptr(), d.shape[0], d.shape[1],
                                                out.data_ptr(), _stream()))
    return out.cpu().numpy().reshape(shape)


def sparsemax(z) -> np.ndarray:
    """Projection of each row onto the simplex (ref numkit.py:42-60)."""
    z = check_finite(z, "sparsemax input")
    d, shape = _rows(z)
    out = torch.empty_like(d)
    _lib.check(_lib.lib().sida_sparsemax_rows_f64(d.data_ptr(), d.shape[0], d.shape[1],
                                                  out.data_ptr(), _stream()))
    return out.cpu().numpy().reshape(shape)


def _topk(z: np.ndarray, k: int) -> np.ndarray:
    d, shape = _rows(z)
    idx = torch.empty((d.shape[0], k), dtype=torch.int64, device=d.device)
    _lib.check(_lib.lib().sida_topk_rows_f64(d.data_ptr(), d.shape[0], d.shape[1], k,
                                             idx.data_ptr(), _stream()))
    return idx.cpu().numpy().reshape(shape[:-1] + (k,))


def topk(z, k: int) -> np.ndarray:
    """Indices of the k largest entries, descending, ties to the lower index
    (ref numkit.py:76-84)."""
    z = check_finite(z, "topk input")
    if z.ndim != 1:
        raise ContractError("topk expects a 1-D vector")
    if not 1 <= k <= z.shape[0]:
        raise ContractError(f"k={k} out of range for length-{z.shape[0]} vector")
    return _topk(z, k)


def topk_rows(z, k: int) -> np.ndarray:
    """Row-wise topk, same ordering contract (ref numkit.py:87-93)."""
    z = check_finite(z, "topk input")
    if not 1 <= k <= z.shape[-1]:
        raise ContractError(f"k={k} out of range for width-{z.shape[-1]} rows")
    return _topk(z, k)
