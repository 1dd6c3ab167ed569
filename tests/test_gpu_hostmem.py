"""Page-locked host memory caches of the drop-in (paper_2503_06322_b200/hostmem.py): results are
identical with and without them, registrations follow their owner's lifetime, pooled result
blocks are reused only after every view of the previous result is gone."""
import gc

import numpy as np
import pytest

import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import hostmem
from paper_2503_06322_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def test_reused_input_registered_and_blobs_identical():
    a = S.smooth_noise((200, 300, 300), seed=5)          # 72 MB: above the registration threshold
    hostmem.enabled = False
    try:
        ref = P.mgard_compress(a, 1e-4)
        ref_out = P.mgard_decompress(ref).values
    finally:
        hostmem.enabled = True
    ev0 = hostmem.alloc_events()
    b1 = P.mgard_compress(a, 1e-4)                        # first sighting: staged
    assert not hostmem._reg.live or all(k[1] != a.ctypes.data for k in hostmem._reg.live)
    b2 = P.mgard_compress(a, 1e-4)                        # second: page-locked, DMA from the array
    assert any(k[1] == a.ctypes.data for k in hostmem._reg.live)
    b3 = P.mgard_compress(a, 1e-4)
    assert b1 == b2 == b3 == ref
    assert hostmem.alloc_events() == ev0 + 1              # one registration, nothing else
    key = next(k for k in hostmem._reg.live if k[1] == a.ctypes.data)
    del a
    gc.collect()
    assert key not in hostmem._reg.live                   # unregistered before numpy freed it

    outs = [P.mgard_decompress(ref).values for _ in range(3)]   # 2nd and 3rd come from the pool
    for o in outs:
        assert np.array_equal(o.view(np.uint8), ref_out.view(np.uint8))
    # three live results: three distinct buffers (a block is never handed out twice)
    assert len({o.ctypes.data for o in outs}) == 3
    view = outs[1][5:]                                    # a view keeps its block checked out
    addr = outs[1].ctypes.data
    del outs
    gc.collect()
    again = [P.mgard_decompress(ref).values for _ in range(2)]
    assert all(o.ctypes.data != addr for o in again)
    assert np.array_equal(view.view(np.uint8), ref_out[5:].view(np.uint8))


def test_fixed_rate_reused_buffers_identical():
    a = S.smooth_noise((160, 256, 512), seed=6)          # 84 MB
    hostmem.enabled = False
    try:
        ref = P.zfp_compress(a, 12)
        ref_out = P.zfp_decompress(ref).values
    finally:
        hostmem.enabled = True
    for _ in range(3):
        assert P.zfp_compress(a, 12) == ref
        assert np.array_equal(P.zfp_decompress(ref).values.view(np.uint8), ref_out.view(np.uint8))


def test_bytes_result_size_hint_paths(oracle):
    """compress -> bytes through the size-hinted, pre-touched result buffer: exact hint, a smaller
    blob (trimmed in place) and a larger blob (fresh allocation) all return the oracle's blob, as an
    exact-length immutable bytes."""
    from paper_2503_06322_b200 import _lib, mgard

    old = _lib.BytesSink.MIN_HINT
    _lib.BytesSink.MIN_HINT = 0
    mgard._SIZE_HINTS.clear()
    try:
        a = S.smooth_noise((60, 70, 80), seed=8)
        ref = oracle.mgard_compress(a, 1e-4)
        for _ in range(3):                                # no hint, then the exact hint
            b = P.mgard_compress(a, 1e-4)
            assert type(b) is bytes and b == ref
        smaller = oracle.mgard_compress(a, 1e-2)          # the hint is keyed by eb_rel: seed it
        big = oracle.mgard_compress(a, 1e-5)
        key = next(iter(mgard._SIZE_HINTS))
        for eb, want in ((1e-2, smaller), (1e-5, big)):
            k = (key[0], key[1], key[2], eb, key[4], key[5])
            mgard._SIZE_HINTS[k] = len(ref)               # hint larger than 1e-2's blob, smaller than 1e-5's
            b = P.mgard_compress(a, eb)
            assert type(b) is bytes and b == want
    finally:
        _lib.BytesSink.MIN_HINT = old


def test_bytes_result_allocation_failure_raises():
    """A failed result allocation (the allocator callback returns NULL) raises AllocationError and
    leaves the context usable (hpdr_mgard_compress_alloc, include/hpdr_b200.h)."""
    from paper_2503_06322_b200 import _lib
    from paper_2503_06322_b200.errors import AllocationError

    a = S.smooth_noise((40, 50, 60), seed=9)
    ref = P.mgard_compress(a, 1e-3)
    orig = _lib.BytesSink._alloc
    _lib.BytesSink._alloc = lambda self, _user, n: None
    try:
        with pytest.raises(AllocationError):
            P.mgard_compress(a, 1e-3)
    finally:
        _lib.BytesSink._alloc = orig
    assert P.mgard_compress(a, 1e-3) == ref
