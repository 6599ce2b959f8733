"""ctypes binding of the sm_100a C ABI (include/sida_b200.h).

This is the only place Python crosses into native code. There is no CPU
fallback: if the library is missing or the device is not an sm_100 part,
``lib()`` raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ContractError, CoverageError, NativeLibraryError, UnservableError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_sida_b200.so")

OK, ERR_CONTRACT, ERR_COVERAGE, ERR_UNSERVABLE, ERR_CUDA, ERR_UNSUPPORTED = range(6)

_vp, _i, _sz = C.c_void_p, C.c_int, C.c_size_t

# name -> (restype, argtypes); mirrors include/sida_b200.h one-to-one.
SIGNATURES = {
    "sida_abi_version": (_i, []),
    "sida_last_error": (C.c_char_p, []),
    "sida_launch_count": (C.c_ulonglong, []),
    "sida_device_check": (_i, [_i]),
    "sida_hash_param_count": (_sz, [_i, _i, _i, _i, _i]),
    "sida_hash_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i, _i, _i]),
    "sida_hash_tables_count": (_sz, [_i, _i, _i, _i, _i]),
    "sida_hash_prepare": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "sida_hash_forward": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i,
                               _i, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sida_debug_hash_prof": (_i, [_vp]),
    "sida_permute_workspace_bytes": (_sz, [_i, _i, _i]),
    "sida_permute_hist": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                               _vp]),
    "sida_gather_rows_bf16": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp]),
    "sida_slot_bytes": (_sz, [_i, _i]),
    "sida_grouped_ffn_bf16": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _vp, _i, _vp, _sz, _i, _vp, _vp,
                                   _vp, _vp, _vp, _vp, _vp, _vp]),
    "sida_debug_gemm_prof": (_i, [_vp]),
    "sida_set_gemm_prof": (_i, [_i]),
    "sida_set_ffn_tiles": (_i, [_i]),
    "sida_get_ffn_tiles": (_i, []),
    "sida_grouped_ffn_f32": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _vp]),
    "sida_combine_ranks": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "sida_gather_bf16_rows": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "sida_unpermute_combine": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "sida_map_combine": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "sida_attention_core": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "sida_out_proj_bytes": (_sz, [_i]),
    "sida_linear_bytes": (_sz, [_i, _i]),
    "sida_embed": (_i, [_vp, _vp, _i, _i, _vp, _vp, _i, _vp, _vp, _vp]),
    "sida_pool_classify": (_i, [_vp, _vp, _i, _i, _vp, _i, _vp, _vp]),
    "sida_linear_bf16": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "sida_out_proj_scatter": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp]),
    "sida_router_topk": (_i, [_vp, _i, _i, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "sida_out_proj_scatter_peer": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _i, _vp,
                                        _vp]),
    "sida_grouped_ffn_bf16_peer": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _vp, _sz, _i, _vp, _vp,
                                        _i, _vp, _vp, _vp]),
    "sida_peer_signal": (_i, [_vp, _i, _i, _i, _vp]),
    "sida_peer_wait": (_i, [_vp, _i, _i, _vp]),
    "sida_segment_map": (_i, [_vp, _vp, _i, _vp, _i, _vp, _vp]),
    "sida_ipc_handle_bytes": (_sz, []),
    "sida_ipc_handle": (_i, [_vp, _vp, C.POINTER(C.c_size_t)]),
    "sida_ipc_open": (_i, [_vp, _sz, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "sida_ipc_close": (_i, [_vp]),
    "sida_softmax_rows_f64": (_i, [_vp, _i, _i, _vp, _vp]),
    "sida_sparsemax_rows_f64": (_i, [_vp, _i, _i, _vp, _vp]),
    "sida_topk_rows_f64": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "sida_router_scores_f64": (_i, [_vp, _i, _i, _vp, _i, _vp, _vp]),
    "sida_moe_token_f64": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp]),
    "sida_expert_copy": (_i, [_vp, _vp, _sz, _vp, _vp, _vp]),
    "sida_poke_i32": (_i, [_vp, _vp, _i, _vp]),
    "sida_copy_sm": (_i, [_vp, _vp, _sz, _vp]),
    "sida_pack_expert_host": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp]),
    "sida_plan_placement": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _i, _vp, _vp]),
}

_lock = threading.Lock()
_handle = None
_device_checked: set[int] = set()


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the library and bind every signature (no device needed)."""
    global _handle
    with _lock:
        if _handle is not None:
            return _handle
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} not found: build it with `python -m paper_2310_18859_b200.build`")
        try:
            h = C.CDLL(path)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _handle = h
        return h


def lib(device: int | None = None) -> C.CDLL:
    """The loaded library, after checking the CUDA device is sm_100 (once per
    device; later calls return at once -- this sits on the per-launch path)."""
    if _handle is not None and _device_checked and device is None:
        return _handle
    h = load()
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the SiDA B200 path has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _device_checked:
        check(h.sida_device_check(dev))
        _device_checked.add(dev)
    return h


def check(status: int) -> None:
    if status == OK:
        return
    msg = (load().sida_last_error() or b"").decode(errors="replace")
    if status == ERR_COVERAGE:
        raise CoverageError(msg)
    if status == ERR_CONTRACT:
        raise ContractError(msg)
    if status == ERR_UNSERVABLE:
        raise UnservableError(msg)
    raise NativeLibraryError(f"[status {status}] {msg}")


def ptr(t) -> int | None:
    """Device/host address of a tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream) -> int:
    return stream.cuda_stream
