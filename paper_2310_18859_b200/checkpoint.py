"""Reference checkpoint containers -> pinned bf16 expert slabs.

Reads and writes the reference's binary container (ref checkpoint.py:1-86):

    magic "SIDAMOE1" | "SIDAHSH1" (8 B), cfg_len uint32, cfg JSON (sorted keys),
    n_tensors uint32, then per tensor: name_len uint16, name, ndim uint8,
    dims ndim x uint64, data prod(dims) x float64 -- all little-endian, C order.

`load_moe` never materialises the float64 model: the file is memory-mapped
and each (layer, expert) slice of w1/b1/w2/b2 is packed straight into its
pinned bf16 slot image by the native packer (sida_pack_expert_host), so a
Switch-base-256 checkpoint (58 GB of float64) streams through a few MB of
host memory into the expert store the residency engine copies from. The
dense tensors (embeddings, mixing attention, routers, head) go to HBM at
bf16 like `MoEModel(config, params=...)`.

`save_moe` writes a model back in the reference's parameter order (ref
moe.py:163-179) from the values the B200 model holds (bf16, widened exactly
to float64), so ref `load_moe` reads it and `load_moe` here round-trips it
bit-exactly. Predictor checkpoints (ref predictor.py:550-571) are float64 on
both sides and round-trip bit-exactly.
"""

from __future__ import annotations

import json
import mmap
import os
import struct
from dataclasses import asdict

import numpy as np
import torch

from .errors import ContractError
from .moe import MoEConfig, MoEModel
from .predictor import PredictorConfig, PredictorNet

MOE_MAGIC = b"SIDAMOE1"
PREDICTOR_MAGIC = b"SIDAHSH1"


# ------------------------------------------------------------------------ container
def _write_header(fh, magic: bytes, config: dict, n_tensors: int) -> None:
    if len(magic) != 8:
        raise ContractError("magic must be exactly 8 bytes")
    cfg = json.dumps(config, sort_keys=True).encode("utf-8")
    fh.write(magic)
    fh.write(struct.pack("<I", len(cfg)))
    fh.write(cfg)
    fh.write(struct.pack("<I", n_tensors))


def _write_tensor_header(fh, name: str, shape) -> None:
    nb = name.encode("utf-8")
    fh.write(struct.pack("<H", len(nb)))
    fh.write(nb)
    fh.write(struct.pack("<B", len(shape)))
    fh.write(struct.pack(f"<{len(shape)}Q", *shape))


def save_container(path, magic: bytes, config: dict, tensors: dict) -> None:
    """ref checkpoint.py:33-51. ``tensors`` values are arrays or callables
    (shape, writer(fh)) for streamed tensors."""
    with open(path, "wb") as fh:
        _write_header(fh, magic, config, len(tensors))
        for name, arr in tensors.items():
            if callable(arr):
                shape, writer = arr()
                _write_tensor_header(fh, name, shape)
                writer(fh)
            else:
                a = np.ascontiguousarray(arr, dtype="<f8")
                _write_tensor_header(fh, name, a.shape)
                fh.write(a.tobytes())


def map_container(path, expected_magic: bytes) -> tuple[dict, dict[str, np.ndarray]]:
    """Parse a container without reading its data: returns (config, name ->
    read-only float64 memmap view), with the reference's checks (bad magic,
    truncation, trailing bytes; ref checkpoint.py:54-86)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ) if size else b""
    off = 0

    def take(n: int) -> bytes:
        nonlocal off
        if off + n > size:
            raise ContractError(f"truncated checkpoint {path}")
        chunk = mm[off:off + n]
        off += n
        return chunk

    magic = take(8)
    if magic != expected_magic:
        raise ContractError(f"bad magic {magic!r} in {path}, expected {expected_magic!r}")
    (cfg_len,) = struct.unpack("<I", take(4))
    config = json.loads(take(cfg_len).decode("utf-8"))
    (n_tensors,) = struct.unpack("<I", take(4))
    tensors: dict[str, np.ndarray] = {}
    for _ in range(n_tensors):
        (name_len,) = struct.unpack("<H", take(2))
        name = take(name_len).decode("utf-8")
        (ndim,) = struct.unpack("<B", take(1))
        dims = struct.unpack(f"<{ndim}Q", take(8 * ndim))
        count = int(np.prod(dims)) if ndim else 1
        if off + 8 * count > size:
            raise ContractError(f"truncated checkpoint {path}")
        tensors[name] = np.frombuffer(mm, dtype="<f8", count=count, offset=off).reshape(dims)
        off += 8 * count
    if off != size:
        raise ContractError(f"trailing bytes in checkpoint {path}")
    return config, tensors


def load_container(path, expected_magic: bytes) -> tuple[dict, dict[str, np.ndarray]]:
    """ref checkpoint.py:54-86: (config, name -> float64 array copies)."""
    config, views = map_container(path, expected_magic)
    return config, {k: np.array(v, dtype=np.float64) for k, v in views.items()}


# ----------------------------------------------------------------------------- MoE
def _moe_names(c: MoEConfig) -> list[tuple[str, tuple]]:
    """Parameter names and shapes in the reference's declared order (ref moe.py:163-179)."""
    d, h, k = c.d_model, c.expert_hidden, c.num_experts
    out = [("tok_emb", (c.vocab_size, d)), ("pos_emb", (c.max_seq_len, d))]
    for layer in range(c.num_layers):
        pre = f"block{layer}."
        out += [(pre + n, (d, d)) for n in ("wq", "wk", "wv", "wo")]
        out += [(pre + "w_r", (d, k)), (pre + "w1", (k, d, h)), (pre + "b1", (k, h)),
                (pre + "w2", (k, h, d)), (pre + "b2", (k, d))]
    out.append(("wc", (d, c.num_classes)))
    return out


def load_moe(path, device=None) -> MoEModel:
    """ref moe.py:587-596, onto the B200 model: dense tensors to HBM at bf16,
    experts packed per (layer, expert) from the memory-mapped file into the
    pinned slot images (never the whole float64 model in host memory)."""
    cfg, tensors = map_container(path, MOE_MAGIC)
    config = MoEConfig(**cfg)
    want = dict(_moe_names(config))
    if set(tensors) != set(want):
        raise ContractError("checkpoint parameter names do not match config")
    for name, arr in tensors.items():
        if tuple(arr.shape) != tuple(want[name]):
            raise ContractError(f"checkpoint tensor {name} has wrong shape")
    return MoEModel(config, params=tensors, device=device)


def _bf16_to_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float32).numpy().astype(np.float64)


def save_moe(model: MoEModel, path) -> None:
    """ref moe.py:581-584 from the values the B200 model holds (bf16 widened
    exactly to float64), streaming the experts slot image by slot image."""
    c = model.config
    d, h, k = c.d_model, c.expert_hidden, c.num_experts
    n2 = 2 * d * h

    def image(layer, e):
        img = model.expert_image(layer, e)[: (n2 + h + d) * 2].view(torch.bfloat16)
        return img.float().numpy().astype("<f8")

    def expert_tensor(layer, part):
        shape = {"w1": (k, d, h), "b1": (k, h), "w2": (k, h, d), "b2": (k, d)}[part]

        def write(fh):
            for e in range(k):
                im = image(layer, e)
                if part == "w1":      # slot holds W1^T (h, d)
                    a = im[: h * d].reshape(h, d).T
                elif part == "w2":    # slot holds W2^T (d, h)
                    a = im[h * d: n2].reshape(d, h).T
                elif part == "b1":
                    a = im[n2: n2 + h]
                else:
                    a = im[n2 + h: n2 + h + d]
                fh.write(np.ascontiguousarray(a, dtype="<f8").tobytes())

        return lambda: (shape, write)

    tensors: dict = {"tok_emb": _bf16_to_f64(model.tok_emb),
                     "pos_emb": _bf16_to_f64(model.pos_emb)}
    for layer in range(c.num_layers):
        pre = f"block{layer}."
        wqkv = _bf16_to_f64(model.wqkv[layer])
        tensors[pre + "wq"], tensors[pre + "wk"], tensors[pre + "wv"] = (
            wqkv[:, :d], wqkv[:, d:2 * d], wqkv[:, 2 * d:])
        tensors[pre + "wo"] = _bf16_to_f64(model.wo[layer])
        tensors[pre + "w_r"] = model.w_r[layer].cpu().numpy().astype(np.float64)
        for part in ("w1", "b1", "w2", "b2"):
            tensors[pre + part] = expert_tensor(layer, part)
    tensors["wc"] = model.wc.cpu().numpy().astype(np.float64)
    save_container(path, MOE_MAGIC, asdict(c), tensors)


# ----------------------------------------------------------------------- predictor
def save_predictor(net: PredictorNet, path) -> None:
    """ref predictor.py:550-557."""
    cfg = asdict(net.config)
    cfg.update(d_model=net.d_model, num_moe_layers=net.num_moe_layers,
               num_experts=net.num_experts)
    save_container(path, PREDICTOR_MAGIC, cfg, net.params)


def load_predictor(path) -> PredictorNet:
    """ref predictor.py:560-571."""
    cfg, tensors = load_container(path, PREDICTOR_MAGIC)
    d_model = cfg.pop("d_model")
    num_moe_layers = cfg.pop("num_moe_layers")
    num_experts = cfg.pop("num_experts")
    net = PredictorNet(PredictorConfig(**cfg), d_model, num_moe_layers, num_experts)
    if set(tensors) != set(net.params):
        raise ContractError("checkpoint parameter names do not match config")
    for name, arr in tensors.items():
        if arr.shape != net.params[name].shape:
            raise ContractError(f"checkpoint tensor {name} has wrong shape")
    net.params = {name: tensors[name] for name in net.params}
    net._packed = {}
    return net


__all__ = ["MOE_MAGIC", "PREDICTOR_MAGIC", "save_container", "load_container", "map_container",
           "load_moe", "save_moe", "load_predictor", "save_predictor"]
