"""Host logic of the multi-GPU paths, on CPU (no GPU needed).

* band partitioning: contiguous, complete, stride-aligned starts (so copy
  anchors never cross a shard, kernels_numba.py:363-373);
* stream partitioning for independent-stream batches;
* the cross-shard reduction of the step's exact partials and the feature
  gather of row-band training, run with world_size 2 over gloo;
* the band slices of a group map reassemble the whole-frame map.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_09339_b200.errors import DataError
from paper_1705_09339_b200.grouping import GroupMap
from paper_1705_09339_b200.parallel import (DistReducer, band_group_map,
                                            band_rows, dist_gather_rows,
                                            streams_for_rank)


@pytest.mark.parametrize("height,parts,stride", [
    (2160, 1, 2), (2160, 2, 2), (2160, 4, 2), (2160, 8, 2), (121, 4, 2),
    (100, 3, 3), (7, 7, 1), (1080, 8, 5), (33, 2, 16)])
def test_band_rows(height, parts, stride):
    rows = band_rows(height, parts, stride)
    assert len(rows) == parts
    assert rows[0][0] == 0 and rows[-1][1] == height
    for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
        assert a1 == b0
    for r0, r1 in rows:
        assert r0 % stride == 0 and r1 > r0
    sizes = [r1 - r0 for r0, r1 in rows[:-1]]
    if sizes:
        assert max(sizes) - min(sizes) <= stride


def test_band_rows_rejects_too_many_parts():
    with pytest.raises(DataError):
        band_rows(4, 3, 2)


@pytest.mark.parametrize("n,world", [(64, 1), (64, 8), (64, 3), (5, 8)])
def test_streams_for_rank(n, world):
    got = [streams_for_rank(n, r, world) for r in range(world)]
    flat = [s for g in got for s in g]
    assert flat == list(range(n))
    assert max(map(len, got)) - min(map(len, got)) <= 1


def test_band_group_map_slices_reassemble():
    rng = np.random.default_rng(0)
    h, w = 10, 6
    gid = rng.integers(-1, 3, size=h * w)
    gm = GroupMap(gid, np.ones((3, 2)), np.ones((3, 2)), np.ones(3),
                  np.bincount(gid[gid >= 0], minlength=3))
    rows = band_rows(h, 3, 2)
    parts = [band_group_map(gm, r0, r1, w).group_id for r0, r1 in rows]
    assert np.array_equal(np.concatenate(parts), gid)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. accum partials: u64 bit patterns in int64, incl. > 2^53 words
        words = 7 * 3 + 1 + 6 * 3 * 2
        rng = np.random.default_rng(100 + rank)
        part = rng.integers(0, 2 ** 40, size=words, dtype=np.int64)
        part[3] = 2 ** 61 + rank          # large fixed-point confidence word
        acc = torch.from_numpy(part.copy())
        DistReducer()(acc)
        # 2. feature gather with unequal bands, in rank (= row) order
        n_rows = [5, 3][rank]
        feats = np.full((n_rows, 2), float(rank)) + np.arange(n_rows)[:, None]
        wfin = np.full(n_rows, 10.0 + rank)
        f_all, w_all = dist_gather_rows()(feats, wfin)
        q.put((rank, acc.numpy().copy(), part, f_all, w_all))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduction_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    want = (res[0][2].astype(np.uint64) + res[1][2].astype(np.uint64))
    for rank, acc, _, f_all, w_all in res:
        assert np.array_equal(acc.astype(np.uint64), want), rank
        assert f_all.shape == (8, 2) and w_all.shape == (8,)
        assert np.array_equal(f_all[:5, 0], np.arange(5.0))
        assert np.array_equal(f_all[5:, 0], 1.0 + np.arange(3.0))
        assert np.array_equal(w_all, [10.0] * 5 + [11.0] * 3)


def test_peer_mailbox_host_side():
    """The host side of the fused row-band sum (cog_peers): struct layout as
    in include/cog_b200.h, mailbox size, the shared step sequence number and
    its parity slots, argument checks -- no GPU work."""
    import ctypes

    from paper_1705_09339_b200 import _lib
    from paper_1705_09339_b200.errors import DataError
    from paper_1705_09339_b200.parallel import PeerMailbox
    lib = _lib.load()
    assert ctypes.sizeof(_lib.Peers) == 16 + 8 * _lib.MAX_RANKS
    words = lib.cog_accum_words(3, 5)
    assert lib.cog_mailbox_words(3, 5, 4) == 2 * 4 * (words + 1)
    assert lib.cog_mailbox_words(3, 5, _lib.MAX_RANKS + 1) == -1
    assert lib.cog_mailbox_words(0, 5, 2) == -1
    box = PeerMailbox(3, 5, 4, 2, [0x1000, 0x2000, 0x3000, 0x4000], fused=True)
    assert box.words == PeerMailbox.size(3, 5, 4)
    seqs = [box.next().seq for _ in range(3)]
    assert seqs == [1, 2, 3] and box.current().seq == 3
    c = box.current()
    assert (c.n_ranks, c.rank) == (4, 2)
    assert [c.mailbox[r] for r in range(4)] == [0x1000, 0x2000, 0x3000, 0x4000]
    with pytest.raises(DataError):
        PeerMailbox(3, 5, 1, 0, [0x1000])
    with pytest.raises(DataError):
        PeerMailbox(3, 5, 3, 0, [0x1000, 0x2000])
    # null mailbox / bad rank / zero sequence number are refused by the C-ABI
    g = _lib.Geom()
    g.total_pixels, g.height, g.width, g.depth = 64, 8, 8, 1
    g.k, g.stride, g.n_groups, g.streams = 3, 2, 0, 1
    bad = _lib.Peers()
    bad.n_ranks, bad.rank, bad.seq = 2, 0, 0
    rc = lib.cog_finalize_p2p(_lib.ref(g), _lib.ref(_lib.Params()),
                              _lib.ref(_lib.State()),
                              ctypes.c_void_p(8), 0, _lib.ref(bad), None)
    assert rc < 0
