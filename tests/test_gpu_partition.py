"""The multi-GPU block partition with the CUDA compressor: two ranks (gloo, both on
GPU 0 of the test box) each compress their dim-0 block through partition.distributed_compress;
the job-wide min/max all-reduce runs inside the library call (RangeExchange / the C ABI's range
hook).  Every rank's blob must equal the oracle's blob of its block under the global range, i.e.
the reference's mgard_compress(block, eb_rel, value_range=global)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from paper_2503_06322_b200 import container as C
from paper_2503_06322_b200 import synthetic as S

pytestmark = pytest.mark.gpu

SHAPE = (97, 66, 129)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    from paper_2503_06322_b200 import partition as PT

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = S.smooth_noise(SHAPE, seed=5)
        lo, hi = C.slab_bounds(SHAPE[0], world, rank)
        block = np.ascontiguousarray(a[lo:hi])
        if mode == "pinned":       # the bench's e2e call: pinned host block, blob into pinned memory
            src = torch.from_numpy(block).pin_memory()
            out = torch.empty(block.nbytes * 2, dtype=torch.uint8).pin_memory()
            n, sizes, vr = PT.distributed_compress(src, 1e-4, out=out)
            blob = bytes(out[:n].numpy())
        elif mode == "device":     # device-resident block (kernel-only leg)
            src = torch.from_numpy(block).cuda()
            blob, sizes, vr = PT.distributed_compress(src, 1e-4)
        else:                      # numpy block
            blob, sizes, vr = PT.distributed_compress(block, 1e-4)
        y = PT.distributed_decompress(blob)
        q.put((rank, blob, sizes, vr, np.asarray(y)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["numpy", "pinned", "device"])
def test_distributed_compress_cuda_two_ranks(mode, oracle):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = S.smooth_noise(SHAPE, seed=5)
    vr = (float(a.min()), float(a.max()))
    for rank, blob, sizes, got_vr, y in res:
        assert got_vr == vr                                   # job-wide range, exchanged in the call
        assert sizes == [len(r[1]) for r in res]              # all-gathered blob sizes
        lo, hi = C.slab_bounds(SHAPE[0], world, rank)
        assert blob == oracle.mgard_compress(np.ascontiguousarray(a[lo:hi]), 1e-4, value_range=vr), rank
        assert np.array_equal(y.view(np.uint8), oracle.mgard_decompress(blob).view(np.uint8))
