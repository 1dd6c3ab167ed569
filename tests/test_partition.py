"""Block partitioning, container format and the multi-rank metadata exchange, on CPU with the
parity oracle as the per-slab compressor (gloo, world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_06322_b200 import container as C
from paper_2503_06322_b200 import partition as PT
from paper_2503_06322_b200 import synthetic as S
from paper_2503_06322_b200.errors import FormatError


def _oracle_compressor(arr, eb, dsz, vr):
    from oracle import oracle as O

    return O.mgard_compress(arr, eb, dsz, value_range=vr)


def _oracle_decompressor(blob):
    from oracle import oracle as O

    return O.mgard_decompress(blob)


def _np_minmax(a):
    return float(a.min()), float(a.max())


def test_container_roundtrip_and_crc():
    h = C.ContainerHeader(0, (4, 5), 1e-3, 4096, -1.0, 2.0,
                          [C.ChunkEntry(0, 10, 0, 3), C.ChunkEntry(10, 10, 0, 5)])
    data = C.write_container(h, [b"abc", b"defgh"])
    h2, p = C.read_container(data)
    assert h2.dims == (4, 5) and [bytes(x) for x in p] == [b"abc", b"defgh"]
    assert [c.payload_offset for c in h2.chunks] == [0, 3]
    empty = C.write_container(C.ContainerHeader(1, (3,), 1e-2, 16, 0.0, 1.0, []), [])
    assert C.read_container(empty)[1] == []
    hdr_len = len(C.header_bytes(h))
    for i in range(hdr_len - 4):
        bad = bytearray(data)
        bad[i] ^= 0x01
        with pytest.raises(FormatError):
            C.read_container(bytes(bad))
    with pytest.raises(FormatError):
        C.read_container(data[:hdr_len + 2])


def test_slab_bounds_tile_exactly():
    for n in (1, 7, 128, 1024):
        for parts in (1, 2, 3, 8):
            if parts > n:
                continue
            b = [C.slab_bounds(n, parts, k) for k in range(parts)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[k][1] == b[k + 1][0] for k in range(parts - 1))


def test_compress_slabs_global_range_and_bound():
    a = S.smooth_noise((24, 20, 18), seed=4)
    data = PT.compress_slabs(a, 1e-3, 3, compressor=_oracle_compressor, minmax=_np_minmax)
    h, payloads = C.read_container(data)
    assert len(payloads) == 3 and (h.vmin, h.vmax) == (float(a.min()), float(a.max()))
    for k, p in enumerate(payloads):
        lo, hi = C.slab_bounds(24, 3, k)
        assert bytes(p) == _oracle_compressor(a[lo:hi], 1e-3, 4096, (h.vmin, h.vmax))
    y = PT.decompress_slabs(data, decompressor=_oracle_decompressor)
    assert np.max(np.abs(y.astype(np.float64) - a)) <= 1e-3 * (h.vmax - h.vmin)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = S.smooth_noise((16, 12, 10), seed=9)
        lo, hi = C.slab_bounds(16, world, rank)
        blob, sizes, vr = PT.distributed_compress(a[lo:hi], 1e-3, compressor=_oracle_compressor, minmax=_np_minmax)
        y = PT.distributed_decompress(blob, decompressor=_oracle_decompressor)
        q.put((rank, blob, sizes, vr, y))
    finally:
        dist.destroy_process_group()


def test_distributed_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = S.smooth_noise((16, 12, 10), seed=9)
    vr = (float(a.min()), float(a.max()))
    for rank, blob, sizes, got_vr, y in res:
        assert got_vr == vr                                   # all-reduced global range
        assert sizes == [len(r[1]) for r in res]              # all-gathered blob sizes
        lo, hi = C.slab_bounds(16, world, rank)
        assert blob == _oracle_compressor(a[lo:hi], 1e-3, 4096, vr)
        assert np.max(np.abs(y.astype(np.float64) - a[lo:hi])) <= 1e-3 * (vr[1] - vr[0])
