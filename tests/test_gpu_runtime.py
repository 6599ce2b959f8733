"""Small-transfer primitives of the serving loop (csrc/runtime.cu):
sida_poke_i32 (int32 rows carried in kernel parameter blocks) and
sida_copy_sm (SM copies to / from pinned host memory). Both stay off the copy
engines, so per-layer slot rows, sequence offsets, token rows and logits do
not queue behind the expert copies."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _h():
    from paper_2310_18859_b200 import _lib

    return _lib, _lib.lib()


@pytest.mark.parametrize("n", [0, 1, 257, 1000, 1001, 2500])
def test_poke_i32_writes_rows_in_stream_order(cuda_device, n):
    import torch

    _l, h = _h()
    st = torch.cuda.Stream()
    dst = torch.full((n + 3,), -7, dtype=torch.int32, device="cuda")
    src = np.arange(n, dtype=np.int32) * 3 - 11
    with torch.cuda.stream(st):
        # an earlier write on the same stream must land first
        dst.fill_(5)
        _l.check(h.sida_poke_i32(dst.data_ptr(), src.ctypes.data, n, st.cuda_stream))
    src[:] = 0  # the values travel in the launch: the host row is free at once
    st.synchronize()
    got = dst.cpu().numpy()
    assert np.array_equal(got[:n], np.arange(n, dtype=np.int32) * 3 - 11)
    assert (got[n:] == 5).all()


def test_poke_i32_contract(cuda_device):
    from paper_2310_18859_b200.errors import ContractError

    _l, h = _h()
    with pytest.raises(ContractError):
        _l.check(h.sida_poke_i32(None, None, 4, None))


@pytest.mark.parametrize("nbytes,off", [(1, 0), (4 * 32768, 0), (4 * 32768 + 12, 4), (2048, 0),
                                        (100003, 1)])
def test_copy_sm_pinned_round_trip(cuda_device, nbytes, off):
    import torch

    _l, h = _h()
    g = np.random.default_rng(nbytes)
    host_src = torch.empty(nbytes + off, dtype=torch.uint8, pin_memory=True)
    host_src.numpy()[:] = g.integers(0, 256, size=nbytes + off, dtype=np.uint8)
    dev = torch.zeros(nbytes + 16, dtype=torch.uint8, device="cuda")
    host_dst = torch.zeros(nbytes + off, dtype=torch.uint8, pin_memory=True)
    st = torch.cuda.Stream()
    _l.check(h.sida_copy_sm(dev.data_ptr() + off, host_src.data_ptr() + off, nbytes,
                            st.cuda_stream))
    _l.check(h.sida_copy_sm(host_dst.data_ptr() + off, dev.data_ptr() + off, nbytes,
                            st.cuda_stream))
    st.synchronize()
    assert torch.equal(dev[off:off + nbytes].cpu(), host_src[off:])
    assert torch.equal(host_dst[off:], host_src[off:])
    assert (dev[:off].cpu() == 0).all() and (dev[off + nbytes:].cpu() == 0).all()
