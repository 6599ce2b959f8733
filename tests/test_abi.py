"""The C-ABI library builds for sm_100a, loads without a GPU and exports
exactly what include/sida_b200.h declares (CPU test: no compute calls)."""

import os
import re
import subprocess

from conftest import REPO

HEADER = os.path.join(REPO, "include", "sida_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(sida_\w+)\s*\(", text, re.M)))


def test_header_lists_the_hot_path_entry_points():
    names = declared()
    for must in ("sida_hash_forward", "sida_permute_hist", "sida_gather_rows_bf16",
                 "sida_grouped_ffn_bf16", "sida_grouped_ffn_f32", "sida_expert_copy",
                 "sida_plan_placement", "sida_combine_ranks"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2310_18859_b200 import _lib

    h = _lib.load()
    for name in declared():
        assert hasattr(h, name), name
    assert set(_lib.SIGNATURES) == set(declared())
    assert h.sida_abi_version() == 1


def test_library_is_sm100a_and_uses_tcgen05_and_tma():
    from paper_2310_18859_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True,
                                       text=True).stdout or "arch = sm_100a" in sass
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA tensor loads
    assert "LDTM" in sass             # tcgen05.ld (TMEM -> registers)


def test_slot_bytes_formula():
    from paper_2310_18859_b200 import _lib

    h = _lib.load()
    assert h.sida_slot_bytes(768, 3072) == (2 * 768 * 3072 + 3072 + 768) * 2  # 9.445 MB
    assert h.sida_slot_bytes(32, 64) % 256 == 0


def test_pack_expert_host_layout():
    import numpy as np
    import torch
    from paper_2310_18859_b200 import _lib

    h = _lib.load()
    d, hh = 64, 128
    g = np.random.default_rng(0)
    w1, b1 = g.normal(size=(d, hh)), g.normal(size=hh)
    w2, b2 = g.normal(size=(hh, d)), g.normal(size=d)
    out = np.zeros(h.sida_slot_bytes(d, hh), dtype=np.uint8)
    arrs = [np.ascontiguousarray(a) for a in (w1, b1, w2, b2)]
    assert h.sida_pack_expert_host(*(a.ctypes.data for a in arrs), d, hh, out.ctypes.data) == 0
    u16 = out.view(np.uint16)

    def bf(a):
        return torch.from_numpy(a).float().bfloat16().view(torch.int16).numpy().view(np.uint16)

    np.testing.assert_array_equal(u16[: hh * d].reshape(hh, d), bf(w1.T.copy()))
    np.testing.assert_array_equal(u16[hh * d : 2 * hh * d].reshape(d, hh), bf(w2.T.copy()))
    np.testing.assert_array_equal(u16[2 * hh * d : 2 * hh * d + hh], bf(b1))
    np.testing.assert_array_equal(u16[2 * hh * d + hh : 2 * hh * d + hh + d], bf(b2))
