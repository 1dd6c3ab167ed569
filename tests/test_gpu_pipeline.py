"""The streams pipeline (HPDR container of per-chunk reference blobs) on the GPU."""
import numpy as np
import pytest

import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import container as CT
from paper_2503_06322_b200 import pipeline as PL
from paper_2503_06322_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,dtype,planes", [((64, 65, 66), np.float32, 16), ((37, 20, 19), np.float64, 5),
                                                 ((300, 41), np.float32, 64), ((5000,), np.float32, 1000)])
def test_pipeline_chunks_are_reference_blobs(shape, dtype, planes, oracle):
    a = S.smooth_noise(shape, seed=7, dtype=dtype)
    data = PL.compress_pipelined(a, 1e-4, chunk_planes=planes)
    h, payloads = CT.read_container(data)
    vr = (float(a.min()), float(a.max()))
    assert (h.vmin, h.vmax) == vr and len(payloads) == -(-shape[0] // planes)
    for c, p in zip(h.chunks, payloads):
        lo = c.raw_offset // (a.size // shape[0])
        hi = lo + c.raw_size // (a.size // shape[0])
        assert bytes(p) == oracle.mgard_compress(a[lo:hi], 1e-4, value_range=vr)
    y = PL.decompress_pipelined(data)
    assert y.dtype == a.dtype and y.shape == a.shape
    assert np.max(np.abs(y.astype(np.float64) - a)) <= 1e-4 * (vr[1] - vr[0])
    ref = np.concatenate([oracle.mgard_decompress(bytes(p)).reshape(-1) for p in payloads]).reshape(shape)
    assert np.array_equal(y.view(np.uint8), ref.view(np.uint8))


def test_pipeline_explicit_schedule_and_trace():
    a = S.smooth_noise((96, 128, 128), seed=2)
    sched = [4, 8, 16, 32, 36]
    data, tr = PL.compress_pipelined(a, 1e-3, chunks=sched, value_range=(-1.0, 2.0), trace=True)
    h, payloads = CT.read_container(data)
    assert [c.raw_size // (128 * 128) for c in h.chunks] == sched
    assert tr.shape == (5, 6) and np.all(tr[:, 1] >= tr[:, 0]) and np.all(tr[:, 3] >= tr[:, 2])
    for k in range(5):   # each chunk: H2D before compute before D2H
        assert tr[k, 2] >= tr[k, 1] - 1e-3 and tr[k, 4] >= tr[k, 3] - 1e-3
    y, tr2 = PL.decompress_pipelined(data, trace=True)
    assert np.max(np.abs(y.astype(np.float64) - a)) <= 1e-3 * 3.0
    assert 0.0 <= PL.overlap_ratio(tr) <= 1.0 and 0.0 <= PL.overlap_ratio(tr2) <= 1.0
    import io

    f = io.StringIO()   # SPEC.md trace export of the real runner's timeline
    assert PL.write_trace_csv(tr, f) == 15
    lines = f.getvalue().splitlines()
    assert lines[0] == ",".join(PL.TRACE_COLUMNS) and all(len(x.split(",")) == 5 for x in lines[1:])
    with pytest.raises(P.ValidationError):
        PL.compress_pipelined(a, 1e-3, chunks=[1, 2, 3])


def test_pipeline_matches_slab_partition_api():
    from paper_2503_06322_b200 import partition as PT

    a = S.smooth_noise((48, 50, 52), seed=4)
    vr = (float(a.min()), float(a.max()))
    via_pipe = PL.compress_pipelined(a, 1e-3, chunk_planes=16)
    via_slabs = PT.compress_slabs(a, 1e-3, 3)
    assert via_pipe == via_slabs
    assert np.array_equal(PT.decompress_slabs(via_pipe), PL.decompress_pipelined(via_slabs))
    h = CT.read_container(via_pipe)[0]
    assert (h.vmin, h.vmax) == vr


def test_pipeline_after_whole_field_call():
    """Regression: chunk plans built while a copy engine streams the next chunk must be visible to
    the compute stream (plan tables were once uploaded on the legacy stream and raced)."""
    import torch

    a = S.smooth_noise((257, 257, 257), seed=0)
    vr = (float(a.min()), float(a.max()))
    P.mgard_compress(torch.from_numpy(a).cuda(), 1e-4)           # whole-field call first
    src = torch.from_numpy(a).pin_memory()
    data = PL.compress_pipelined(src, 1e-4, value_range=vr, chunk_planes=63)
    assert data == PL.compress_pipelined(a, 1e-4, value_range=vr, chunk_planes=63)
    y = PL.decompress_pipelined(data)
    assert np.max(np.abs(y.astype(np.float64) - a)) <= 1e-4 * (vr[1] - vr[0])


def test_relative_pipeline_equals_known_range():
    """Relative mode (range found on the device while chunks decompose) == the same run with the
    range given up front: byte-identical containers."""
    a = S.grf((96, 70, 66), m=4, seed=5)
    rel = PL.compress_pipelined(a, 1e-3, chunk_planes=20)
    known = PL.compress_pipelined(a, 1e-3, chunk_planes=20, value_range=(float(a.min()), float(a.max())))
    assert rel == known


def test_relative_pipeline_non_finite_raises():
    a = S.smooth_noise((40, 33, 31), seed=6)
    a[17, 3, 4] = np.nan
    with pytest.raises(P.ValidationError):
        PL.compress_pipelined(a, 1e-3, chunk_planes=8)


def test_adaptive_pipeline_profiles_and_tiles(oracle):
    """Algorithm 4 end to end: Φ profiled on the device, Θ from a pinned copy, the schedule tiles
    dim 0 and every chunk is a reference blob."""
    a = S.smooth_noise((200, 64, 64), seed=8)
    phi, theta, samples = PL.profile_models(a, 1e-3, sizes_mb=(1, 2, 4))
    assert len(samples) == 3 and phi.gamma > 0 and theta.beta_copy > 0
    vr = (float(a.min()), float(a.max()))
    data = PL.compress_adaptive(a, 1e-3, value_range=vr, models=(phi, theta), c_init=1 << 20)
    h, payloads = CT.read_container(data)
    assert sum(c.raw_size for c in h.chunks) == a.size
    plane = a.size // a.shape[0]
    for c, p in zip(h.chunks, payloads):
        lo = c.raw_offset // plane
        assert bytes(p) == oracle.mgard_compress(a[lo:lo + c.raw_size // plane], 1e-3, value_range=vr)
