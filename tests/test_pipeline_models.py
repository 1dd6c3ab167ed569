"""Chunk-size models of the pipeline (hpdr/pipeline/models.py; SPEC.md:430-491 examples) and
the overlap metric.  CPU only."""
import numpy as np
import pytest

from paper_2503_06322_b200 import pipeline as PL
from paper_2503_06322_b200.errors import ValidationError

MB = 1 << 20


def test_next_chunk_size_spec_examples():
    # Φ saturated with γ·β_copy = 1: chunk size stable
    beta = 1.0 / (10e9)
    m = PL.ThroughputModel.saturated(10e9)
    t = PL.TransportModel(beta)
    assert PL.next_chunk_size(16 * MB, m, t, 1 << 40, 1 << 40) == 16 * MB
    # γ·β = 0.5: compute twice as slow as copy -> doubles until the limit
    m2 = PL.ThroughputModel.saturated(5e9)
    assert PL.next_chunk_size(16 * MB, m2, PL.TransportModel(1.0 / 10e9), 1 << 40, 1 << 40) == 32 * MB
    assert PL.next_chunk_size(16 * MB, m2, PL.TransportModel(1.0 / 10e9), 20 * MB, 1 << 40) == 20 * MB
    # clamped to the remaining size, never 0 unless nothing remains
    assert PL.next_chunk_size(16 * MB, m, t, 1 << 40, 3 * MB) == 3 * MB
    assert PL.next_chunk_size(16 * MB, m, t, 1 << 40, 0) == 0
    assert PL.next_chunk_size(1, m, t, 1 << 40, 100, slab_bytes=7) == 7
    with pytest.raises(ValidationError):
        PL.next_chunk_size(0, m, t, 10, 10)


def test_fit_recovers_noiseless_model():
    alpha, beta, gamma = 40.0, 1e8, 8e9
    c_thr = (gamma - beta) / alpha
    sizes = [c_thr * f for f in (0.2, 0.3, 0.45, 0.6, 0.8, 1.2, 2.0, 4.0)]
    prof = [(c, alpha * c + beta if c < c_thr else gamma) for c in sizes]
    m = PL.fit_throughput_model(prof)
    assert abs(m.gamma - gamma) / gamma < 1e-9
    assert abs(m.alpha - alpha) / alpha < 1e-6 and abs(m.c_threshold - c_thr) / c_thr < 1e-6
    sat = PL.fit_throughput_model([(1e6, 5e9), (2e6, 5e9), (4e6, 5e9)])
    assert sat.alpha == 0.0 and sat.phi(123) == 5e9
    with pytest.raises(ValidationError):
        PL.fit_throughput_model([(1, 1), (2, 2)])
    with pytest.raises(ValidationError):
        PL.fit_throughput_model([(1, 1), (1, 2), (1, 3)])


def test_transport_ema():
    t = PL.TransportModel(1e-9)
    t.observe(1000, 2e-6)
    assert abs(t.beta_copy - (1e-9 + 0.25 * (2e-9 - 1e-9))) < 1e-24
    t.observe(0, 1.0)
    with pytest.raises(ValidationError):
        PL.TransportModel(0.0)


def test_adaptive_schedule_tiles_and_grows():
    plane = 4 * MB
    m = PL.ThroughputModel.saturated(5e9)          # compute 2x slower than the copy
    t = PL.TransportModel(1.0 / 10e9)
    sched = PL.adaptive_schedule(256, plane, m, t, c_init=16 * MB, c_limit=256 * MB)
    assert sum(sched) == 256 and all(s > 0 for s in sched)
    assert sched[:4] == [4, 8, 16, 32]              # doubling (Algorithm 4 with γβ = 0.5)
    assert max(sched) <= 64
    flat = PL.adaptive_schedule(100, plane, PL.ThroughputModel.saturated(10e9), t, c_init=16 * MB)
    assert set(flat[:-1]) == {4}


def test_overlap_ratio_spec_examples():
    # copy [0,2) with compute [1,3): 0.5
    tr = np.array([[0, 2, 1, 3, 3, 3]], float)
    assert PL.overlap_ratio(tr) == pytest.approx(0.5)
    serial = np.array([[0, 1, 1, 2, 2, 3]], float)
    assert PL.overlap_ratio(serial) == 0.0
    inside = np.array([[1, 2, 0, 5, 3, 4]], float)
    assert PL.overlap_ratio(inside) == 1.0
    assert PL.overlap_ratio(np.zeros((0, 6))) == 0.0


def test_container_headers_round_trip_and_reject_corruption():
    """HPDR container for both reducers: header bytes round-trip, a flipped header
    byte fails the CRC, an unknown pipeline id and truncation raise FormatError."""
    from paper_2503_06322_b200 import container as CT
    from paper_2503_06322_b200.errors import FormatError

    pays = [b"abc", b"", b"defgh"]
    for h in (CT.ContainerHeader(0, (9, 4, 5), 1e-3, 4096, -1.0, 2.0,
                                 [CT.ChunkEntry(0, 40, 0, 3), CT.ChunkEntry(40, 80, 0, 0), CT.ChunkEntry(120, 60, 0, 5)]),
              CT.ContainerHeader(1, (9, 20), 0.0, 0, 0.0, 0.0,
                                 [CT.ChunkEntry(0, 60, 0, 3), CT.ChunkEntry(60, 60, 0, 0), CT.ChunkEntry(120, 60, 0, 5)],
                                 pipeline=CT.PIPELINE_ZFP, rate=17)):
        data = CT.write_container(h, pays)
        h2, p2 = CT.read_container(data)
        assert (h2.pipeline, h2.dtype, h2.dims, h2.rate) == (h.pipeline, h.dtype, h.dims, h.rate)
        assert [bytes(p) for p in p2] == pays
        if h.pipeline == CT.PIPELINE_MGARD:
            assert (h2.eb_rel, h2.dict_size, h2.vmin, h2.vmax) == (1e-3, 4096, -1.0, 2.0)
        bad = bytearray(data)
        bad[12] ^= 1
        with pytest.raises(FormatError):
            CT.read_container(bytes(bad))
        bad = bytearray(data)
        bad[6] = 0
        with pytest.raises(FormatError):
            CT.read_container(bytes(bad))
        with pytest.raises(FormatError):
            CT.read_container(data[:-1])


def test_trace_csv_export_spec_columns(tmp_path):
    """SPEC.md External Interfaces: CSV (task_kind, chunk_id, queue, start_ns, end_ns)."""
    import csv

    tr = np.array([[0.0, 1.0, 1.0, 3.0, 3.0, 4.0],
                   [1.0, 2.0, 3.0, 5.0, 5.0, 6.0],
                   [2.0, 3.0, 5.0, 7.0, 7.0, 8.0],
                   [3.0, 4.0, 7.0, 9.0, 9.0, 10.0]])
    p = tmp_path / "trace.csv"
    assert PL.write_trace_csv(tr, str(p)) == 12
    rows = list(csv.reader(open(p)))
    assert tuple(rows[0]) == PL.TRACE_COLUMNS
    body = [(r[0], int(r[1]), int(r[2]), int(r[3]), int(r[4])) for r in rows[1:]]
    assert sorted({r[0] for r in body}) == ["COMPUTE", "D2H", "H2D"]
    assert all(q == k % 3 for _, k, q, _, _ in body)                       # round-robin queues
    assert ("COMPUTE", 1, 1, 3_000_000, 5_000_000) in body                  # ms -> ns, origin at 0
    assert [r[3] for r in body] == sorted(r[3] for r in body)
    # the CSV is the same timeline overlap_ratio measures
    back = np.zeros_like(tr)
    col = {"H2D": 0, "COMPUTE": 2, "D2H": 4}
    for kind, k, _, a, b in body:
        back[k, col[kind]], back[k, col[kind] + 1] = a / 1e6, b / 1e6
    assert PL.overlap_ratio(back) == pytest.approx(PL.overlap_ratio(tr))
    assert PL.write_trace_csv(np.zeros((0, 6)), str(tmp_path / "empty.csv")) == 0
