"""Expert-parallel host logic: split sizes and the regroup map
against brute force, and the transport over a world_size-2 gloo group on CPU.
The GPU data path with real kernels is tests/test_gpu_expert_parallel.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_18859_b200.errors import ContractError
from paper_2310_18859_b200.expert_parallel import GlooTransport, ep_regroup, ep_splits


def _brute(counts, layer, rank, world):
    K = counts.shape[2]
    kl = K // world
    # receive buffer: for each source g, its rows for my experts, expert ascending
    recv = [(g, e) for g in range(world) for e in range(rank * kl, (rank + 1) * kl)
            for _ in range(counts[g, layer, e])]
    order = sorted(range(len(recv)), key=lambda i: (recv[i][1], recv[i][0], i))
    return np.array(order, dtype=np.int32)


@pytest.mark.parametrize("world,K", [(2, 8), (4, 8), (8, 128), (1, 4)])
def test_splits_and_regroup_match_brute_force(world, K):
    g = np.random.default_rng(world * K)
    L = 3
    counts = g.integers(0, 6, size=(world, L, K))
    counts[0, 1, :] = 0  # a rank that routes nothing in one layer
    for rank in range(world):
        for layer in range(L):
            send, recv = ep_splits(counts, layer, rank, world)
            kl = K // world
            assert send.sum() == counts[rank, layer].sum()
            for r2 in range(world):  # what r2 receives from me == what I send to r2
                assert ep_splits(counts, layer, r2, world)[1][rank] == send[r2]
            src, off = ep_regroup(counts, layer, rank, world)
            np.testing.assert_array_equal(src, _brute(counts, layer, rank, world))
            assert off[-1] == recv.sum() == src.size
            np.testing.assert_array_equal(np.diff(off),
                                          counts[:, layer, rank * kl:(rank + 1) * kl].sum(0))


def test_uneven_expert_split_is_rejected():
    with pytest.raises(ContractError):
        ep_splits(np.zeros((3, 1, 8), dtype=np.int64), 0, 0, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _transport_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = GlooTransport()
        hist = torch.full((2, 4), rank, dtype=torch.int32)
        allh = tr.all_gather(hist)
        assert allh.shape == (world, 2, 4) and int(allh[1, 0, 0]) == 1
        # rank r sends (r+1)*(g+1) rows to rank g; rows carry (src, dst, i) in bf16 bits
        send_rows = [(rank + 1) * (g + 1) for g in range(world)]
        recv_rows = [(g + 1) * (rank + 1) for g in range(world)]
        rows = []
        for g in range(world):
            for i in range(send_rows[g]):
                rows.append([rank, g, i, 0])
        send = torch.tensor(rows, dtype=torch.float32).to(torch.bfloat16)
        recv = tr.all_to_all(send, send_rows, recv_rows)
        assert recv.dtype == torch.bfloat16
        got = recv.float().numpy()
        pos = 0
        for g in range(world):
            for i in range(recv_rows[g]):
                assert list(got[pos][:3]) == [g, rank, i]
                pos += 1
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_gloo_transport_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}


def _seg_map(start, val, n_seg, index):
    """Host mirror of sida_segment_map."""
    out = np.empty(len(index), dtype=np.int64)
    for i, p in enumerate(index):
        b = int(np.searchsorted(start[:n_seg], p, side="right")) - 1
        out[i] = val[b] + p - start[b]
    return out


@pytest.mark.parametrize("world,K,L", [(2, 8, 2), (4, 8, 3), (8, 64, 1), (1, 4, 2)])
def test_peer_maps_round_trip(world, K, L):
    """Dispatch then return (ep_peer_maps, as sida_segment_map applies them)
    bring every source row back to its own expert-sorted position, and each
    owner's receive buffer is expert-major / source-minor like ep_regroup."""
    from paper_2310_18859_b200.expert_parallel import ep_peer_maps

    g = np.random.default_rng(world + K + L)
    counts = g.integers(0, 5, size=(world, L, K))
    counts[-1, 0, :] = 0
    sx, sy = 10_000, 1_000
    kl = K // world
    for layer in range(L):
        maps = [ep_peer_maps(counts, layer, r, world, sx, sy) for r in range(world)]
        filled = {}
        for src in range(world):
            d_start, d_val, *_ = maps[src]
            n = int(counts[src, layer].sum())
            dst = _seg_map(d_start, d_val, K, np.arange(n))
            for p, v in enumerate(dst):
                q, row = divmod(int(v), sx)
                e = int(np.searchsorted(d_start, p, side="right")) - 1
                assert q == e // kl
                assert (q, row) not in filled
                filled[(q, row)] = (src, p, e)
        for q in range(world):
            _, _, r_start, r_val, off_l, n_recv = maps[q]
            assert sorted(r for (qq, r) in filled if qq == q) == list(range(n_recv))
            back = _seg_map(r_start, r_val, kl * world, np.arange(n_recv))
            keys = [filled[(q, j)] for j in range(n_recv)]
            # expert-major, source-minor, each source's rows in its own order
            assert keys == sorted(keys, key=lambda t: (t[2], t[0], t[1]))
            for j, v in enumerate(back):
                src, pos = divmod(int(v), sy)
                assert (src, pos) == keys[j][:2]
            assert off_l[-1] == n_recv


@pytest.mark.parametrize("world,K,L,chunks", [(2, 8, 2, 2), (4, 8, 2, 3), (8, 128, 1, 2),
                                              (1, 4, 2, 1), (2, 128, 1, 4)])
def test_chunked_layer_plan_round_trip(world, K, L, chunks):
    """The chunked NCCL path's maps (ep_layer_plan, applied like
    sida_segment_map / all_to_all_single / the FFN row_map would): each
    chunk's exchange delivers every row to its owner, the regrouped rows are
    expert-major / source-minor (ep_regroup's order within the chunk), and the
    return exchange lands each row back at the dispatch position its source
    sent it from (the position sida_map_combine reads)."""
    from paper_2310_18859_b200.expert_parallel import ep_layer_plan

    g = np.random.default_rng(world * 7 + K + chunks)
    counts = g.integers(0, 5, size=(world, L, K))
    counts[0, 0, :K // 2] = 0
    kl = K // world
    for layer in range(L):
        plans = [ep_layer_plan(counts, layer, r, world, chunks) for r in range(world)]
        # each source's rows tagged (src, x_perm position, expert), placed by dmap
        sends = []
        for r, p in enumerate(plans):
            n = int(counts[r, layer].sum())
            dmap = _seg_map(p["d_start"].astype(np.int64), p["d_val"], K, np.arange(n))
            assert sorted(dmap.tolist()) == list(range(n))
            buf = [None] * n
            for pos in range(n):
                e = int(np.searchsorted(p["d_start"], pos, side="right")) - 1
                buf[dmap[pos]] = (r, pos, e)
            sends.append(buf)
        n_chunks = len(plans[0]["chunks"])
        backs = [[None] * len(s) for s in sends]
        for ci in range(n_chunks):
            # all_to_all_single of chunk ci
            recvs = []
            for q in range(world):
                parts = []
                for src in range(world):
                    ch = plans[src]["chunks"][ci]
                    cs0 = plans[src]["chunk_start"][ci]
                    off = cs0 + sum(ch["send_rows"][:q])
                    parts += sends[src][off:off + ch["send_rows"][q]]
                assert len(parts) == sum(plans[q]["chunks"][ci]["recv_rows"])
                recvs.append(parts)
            for q in range(world):
                ch = plans[q]["chunks"][ci]
                e0, e1 = ch["experts"]
                n = ch["n_recv"]
                src_map = _seg_map(ch["seg_start"].astype(np.int64), ch["seg_val"],
                                   (e1 - e0) * world, np.arange(n))
                x_loc = [recvs[q][j] for j in src_map]
                assert all(q * kl + e0 <= t[2] < q * kl + e1 for t in x_loc)
                assert x_loc == sorted(x_loc, key=lambda t: (t[2], t[0], t[1]))
                assert np.diff(ch["off_local"]).tolist() == \
                    counts[:, layer, q * kl + e0:q * kl + e1].sum(0).tolist()
                # FFN writes x_loc row j back to receive position src_map[j]
                ret = [None] * n
                for j, v in enumerate(src_map):
                    ret[v] = x_loc[j]
                # return all_to_all: recv_rows / send_rows swapped
                pos = 0
                for src in range(world):
                    cnt = ch["recv_rows"][src]
                    chs = plans[src]["chunks"][ci]
                    at = plans[src]["chunk_start"][ci] + sum(chs["send_rows"][:q])
                    backs[src][at:at + cnt] = ret[pos:pos + cnt]
                    pos += cnt
        for r in range(world):
            assert backs[r] == sends[r]
