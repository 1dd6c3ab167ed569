"""Parity of the CUDA path against the reference (golden vectors from the reference itself)
and the C oracle, through the public API / C ABI.  Needs a B200: run with -m gpu."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import huffman as PH
from paper_2503_06322_b200 import synthetic as S
from paper_2503_06322_b200.errors import CorruptStreamError, ValidationError

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_small_blobs_match_reference(small_cases):
    for c in small_cases:
        vr = tuple(c["value_range"]) if c["value_range"] else None
        blob = P.mgard_compress(c["input"], c["eb_rel"], c["dict_size"], value_range=vr)
        assert blob == c["blob"], (c["i"], c["shape"], len(blob), len(c["blob"]))


def test_small_decompress_matches_reference(small_cases):
    for c in small_cases:
        out = P.mgard_decompress(c["blob"])
        assert out.values.dtype == c["out"].dtype
        assert np.array_equal(out.values.view(np.uint8), c["out"].view(np.uint8)), c["i"]


def test_decompose_recompose_bit_exact(small_cases):
    for c in small_cases:
        cs = P.decompose(c["input"])
        assert np.array_equal(cs.values.view(np.uint64), c["coef"].view(np.uint64)), c["i"]
        rec = P.recompose(P.CoefficientSet(c["coef"].shape, c["coef"], [], 0.0, 0.0))
        assert np.array_equal(rec.view(np.uint64), c["recomp"].view(np.uint64)), c["i"]


def test_quantize_dequantize_match_oracle(small_cases, oracle):
    for c in small_cases[:20]:
        coef = c["coef"]
        u_min, u_max = float(c["input"].min()), float(c["input"].max())
        vr = tuple(c["value_range"]) if c["value_range"] else None
        q = P.quantize(P.CoefficientSet(coef.shape, coef, [], u_min, u_max), None, c["eb_rel"], c["dict_size"], vr)
        o = oracle.quantize(coef, u_min, u_max, c["eb_rel"], c["dict_size"], vr)
        assert np.array_equal(q.keys, o["keys"]), c["i"]
        assert np.array_equal(q.outlier_idx, o["outlier_idx"]) and np.array_equal(q.outlier_bins, o["outlier_bins"])
        assert np.array_equal(q.coarse_values.view(np.uint64), o["coarse_values"].view(np.uint64))
        assert q.bin_width == o["bin_width"] and q.eb_abs == o["eb_abs"]
        d = P.dequantize(q)
        ref = np.unique  # noqa: F841
        back = d.values.reshape(-1)
        bins = (q.keys.astype(np.int64) >> 1) ^ -(q.keys.astype(np.int64) & 1)
        exp = bins.astype(np.float64) * q.bin_width
        exp[q.outlier_idx.astype(np.int64)] = q.outlier_bins.astype(np.float64) * q.bin_width
        hidx = P.build_hierarchy(coef.shape).coarsest_flat_indices().astype(np.int64)
        exp[hidx] = q.coarse_values
        assert np.array_equal(back.view(np.uint64), exp.view(np.uint64)), c["i"]


def test_huffman_streams_match_reference(huffman_golden):
    meta, data = huffman_golden
    for i, m in enumerate(meta["streams"]):
        keys = data[f"keys{i}"]
        s = PH.huffman_compress(keys, m["dict_size"])
        assert s == data[f"stream{i}"].tobytes(), m["name"]
        back = PH.huffman_decompress(data[f"stream{i}"].tobytes())
        assert np.array_equal(back, keys), m["name"]
        h = PH.histogram(keys, m["dict_size"])
        assert np.array_equal(h.counts, np.bincount(keys, minlength=m["dict_size"]))


def test_corrupt_streams_match_reference(corrupt_cases):
    for name, c in corrupt_cases.items():
        blob = bytes.fromhex(c["hex"])
        if c["ok"]:
            out = P.mgard_decompress(blob).values
            assert hashlib.sha256(out.tobytes()).hexdigest() == c["sha"], name
            continue
        exc = {"CorruptStreamError": CorruptStreamError, "ValidationError": ValidationError,
               "OverflowError": OverflowError, "IndexError": IndexError, "ValueError": ValueError}[c["exc"]]
        with pytest.raises(exc) as ei:
            P.mgard_decompress(blob)
        assert type(ei.value) is exc or c["exc"] == "ValueError", (name, type(ei.value))
        if c["exc"] == "CorruptStreamError":
            assert ei.value.bit_offset == c["bit_offset"], (name, ei.value.bit_offset)


def test_random_shapes_vs_oracle(oracle):
    rng = np.random.default_rng(11)
    for t in range(40):
        rank = int(rng.integers(1, 5))
        dims = tuple(int(rng.integers(1, {1: 3000, 2: 90, 3: 40, 4: 14}[rank])) for _ in range(rank))
        dt = np.float32 if t % 2 else np.float64
        a = (rng.random(dims) * rng.choice([1.0, 1e3, 1e-3])).astype(dt)
        if t % 5 == 0:
            a = S.smooth_noise(dims, seed=t, dtype=dt)
        eb = float(rng.choice([1e-2, 1e-3, 1e-4, 1e-5]))
        dsz = int(rng.choice([4096, 4096, 256, 65535, 16]))
        blob = P.mgard_compress(a, eb, dsz)
        ref = oracle.mgard_compress(a, eb, dsz)
        assert blob == ref, (dims, dt, eb, dsz)
        out = P.mgard_decompress(blob).values
        assert np.array_equal(out.view(np.uint8), oracle.mgard_decompress(blob).view(np.uint8))


def test_error_bound_and_abs_api():
    a = S.grf((65, 66, 67), m=4, seed=3)
    for e in (1e-1, 1e-3, 3.0):
        blob = P.compress(a, e, norm="linf", mode="abs")
        y = P.decompress(blob)
        assert float(np.max(np.abs(y.astype(np.float64) - a.astype(np.float64)))) <= e
        assert np.frombuffer(blob[1 + 24 + 29:1 + 24 + 37], "<f8")[0] == e   # stored eb_abs == e exactly
    blob = P.compress(a, 1e-3, norm="l2", mode="rel")
    y = P.decompress(blob)
    rng_ = float(a.max()) - float(a.min())
    assert float(np.max(np.abs(y.astype(np.float64) - a))) <= 1e-3 * rng_


def test_validation_errors():
    a = np.zeros((8, 8), np.float32)
    with pytest.raises(ValidationError):
        P.mgard_compress(a, 1.5)
    with pytest.raises(ValidationError):
        P.mgard_compress(a, 1e-3, dict_size=1)
    with pytest.raises(ValidationError):
        P.mgard_compress(np.zeros((4, 4), np.int32), 1e-3)
    b = a.copy()
    b[3, 3] = np.nan
    with pytest.raises(ValidationError):
        P.mgard_compress(b, 1e-3)
    with pytest.raises(ValidationError):   # bin overflow: tiny range, huge coefficient
        P.mgard_compress(np.array([0.0, 1e300, 0.0, 1.0], np.float64), 1e-3, value_range=(0.0, 1e-300))
    with pytest.raises(ValidationError):
        PH.histogram(np.array([5], np.uint32), 4)


def test_context_cache_no_realloc():
    cache = P.ContextCache()
    a = S.smooth_noise((33, 34, 35), seed=1)
    b1 = P.mgard_compress(a, 1e-3, cache=cache)
    ev = cache.total_alloc_events
    for _ in range(5):
        assert P.mgard_compress(a, 1e-3, cache=cache) == b1
    assert cache.total_alloc_events == ev
    P.mgard_compress(a, 1e-4, cache=cache)
    assert len(cache) == 2


def test_device_buffers_in_place():
    torch = pytest.importorskip("torch")
    a = S.smooth_noise((40, 41, 42), seed=2)
    ref = P.mgard_compress(a, 1e-4)
    t = torch.from_numpy(a).cuda()
    assert P.mgard_compress(t, 1e-4) == ref
    pin = torch.from_numpy(a).pin_memory()
    assert P.mgard_compress(pin, 1e-4) == ref
    out = torch.empty(a.shape, dtype=torch.float32, device="cuda")
    P.mgard_decompress(ref, out=out)
    assert np.array_equal(out.cpu().numpy(), P.decompress(ref))


def test_config_c1_matches_reference_hash():
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["C1_grf129_abs1e-3"]
    a = S.grf((129,) * 3, m=8, seed=0)
    assert S.sha256(a) == cfg["input_sha"], "input generator differs on this host"
    blob = P.mgard_compress(a, 1e-3, value_range=(0.0, 1.0))
    assert hashlib.sha256(blob).hexdigest() == cfg["blob_sha"]
    out = P.mgard_decompress(blob).values
    assert S.sha256(out) == cfg["out_sha"]


@pytest.mark.slow
def test_config_c2_c3_c4_match_reference_hash():
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))
    cases = [("C2_smooth513_rel1e-4", lambda: S.smooth_noise((513,) * 3, seed=0))]
    for f in S.NYX_FIELDS[:3] + ("velocity_x",):
        for eb in ("0.01", "1e-05"):
            cases.append((f"C3_{f}_129_{eb}", lambda f=f: S.nyx_like((129,) * 3, f)))
    cases.append(("C3_temperature_512_1e-3", lambda: S.nyx_like((512,) * 3, "temperature")))
    for name, gen in cases:
        if name not in cfg:
            continue
        c = cfg[name]
        a = gen()
        assert S.sha256(a) == c["input_sha"], name
        vr = tuple(c["value_range"]) if c["value_range"] else None
        blob = P.mgard_compress(a, c["eb_rel"], value_range=vr)
        assert len(blob) == c["blob_len"] and hashlib.sha256(blob).hexdigest() == c["blob_sha"], name
        out = P.mgard_decompress(blob).values
        assert S.sha256(out) == c["out_sha"], name


_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2503_06322_b200 as P
from oracle import oracle as O
from paper_2503_06322_b200 import synthetic as S
import torch
cases = [((33, 34, 35), np.float32), ((16, 5, 7), np.float32), ((65, 40), np.float32), ((1000,), np.float32),
         ((12, 10, 9), np.float32), ((40, 36, 64), np.float32), ((67, 20, 34), np.float64), ((9, 48, 16), np.float64),
         ((70, 66, 90), np.float32)]   # (last: coarse grid above the one-block solve; streamed plane-axis solve)
for shape, dt in cases:
    a = S.smooth_noise(shape, seed=3, dtype=dt)
    for vr in (None, (-1.0, 2.0)):
        bd = P.mgard_compress(torch.from_numpy(a).cuda(), 1e-3, value_range=vr)
        assert bd == O.mgard_compress(a, 1e-3, value_range=vr), (shape, vr, "device input")
        b = P.mgard_compress(a, 1e-3, value_range=vr)
        assert b == O.mgard_compress(a, 1e-3, value_range=vr), (shape, vr)
        y = P.mgard_decompress(b).values
        assert np.array_equal(y.view(np.uint8), O.mgard_decompress(b).view(np.uint8)), shape
print("variant ok")
"""


@pytest.mark.parametrize("env", [{"HPDR_GENERIC": "1"}, {"HPDR_NO_STREAM": "1"}, {"HPDR_NO_QUAD": "1"},
                                 {"HPDR_NO_TMA": "1"}, {"HPDR_QUAD_SLABS": "3"}, {"HPDR_QUAD_SLABS": "64"}, {"HPDR_QUAD_MIN": "0"},
                                 {"HPDR_NO_TINY": "1"}, {"HPDR_NO_TINY": "1", "HPDR_NO_GRAPH": "1"},
                                 {"HPDR_NO_PLANE_SPLIT": "1"}, {"HPDR_NO_QUAD_FINAL": "1"}, {"HPDR_NO_QUAD_P1R": "1"},
                                 {"HPDR_NO_STREAM_L1": "1", "HPDR_STREAM_DECODE_MIN_BITS": "0"},
                                 {"HPDR_STREAM_DECODE_MIN_BITS": "0"}, {"HPDR_QF_COLUMNS": "1"}, {"HPDR_P2_ONE_COL": "1"},
                                 {"HPDR_THOMAS_TILE": "1"}, {"HPDR_NO_FWD_STREAM": "1"}, {"HPDR_NO_DEFER_L1": "1"},
                                 {"HPDR_STREAM_DECODE_MIN_BITS": "0", "HPDR_DEC_GROUPS": "32"}, {}])
def test_execution_variants_bit_identical(env):
    """Every execution variant gives the reference's blobs: the per-axis (generic) path, the non-streamed
    fused path, pass 1 without quads, the quad kernel without TMA, forced slab splits (down to two coarse
    planes per slab), the shared-memory tile Thomas solve at every size, and the small end of the
    hierarchy as per-level launches instead of the one-block kernel (tiny.cu), and the finest
    correction solved whole before the output slabs instead of plane range by plane range, and the
    final level with one node per thread instead of quads, and the finest plane-axis solve run whole
    after the last chunk instead of following its right-hand side."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT % root], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stderr[-2000:]


def test_thomas_fast_division_matches_ieee():
    """The Thomas back substitution's verified fast division never differs from __ddiv_rn."""
    import ctypes as C

    from paper_2503_06322_b200._lib import check, lib

    m, f = C.c_uint64(), C.c_uint64()
    check(lib().hpdr_selftest_div(1 << 26, 12345, C.byref(m), C.byref(f)))
    assert m.value == 0
    assert f.value < (1 << 26) // 1000   # the exact redo is rare


@pytest.mark.parametrize("flip", [None, 0.37, 0.81])
def test_streamed_decompress_matches_oracle(flip, oracle):
    """Blobs with a >= 4 MB payload take the streamed decompress (payload in unit groups, the finest
    correction slab by slab); it must reproduce the reference bit for bit, corrupted payloads included."""
    a = S.smooth_noise((257, 257, 257), seed=3)
    blob = bytearray(P.mgard_compress(a, 1e-4))
    if flip is not None:   # a payload bit (the stream tail is the packed payload)
        pos = int(len(blob) * flip)
        blob[pos] ^= 0x10
    blob = bytes(blob)
    try:
        want = oracle.mgard_decompress(blob)
    except Exception as e:   # noqa: BLE001
        with pytest.raises(type(e)):
            P.mgard_decompress(blob)
        return
    got = P.mgard_decompress(blob).values
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_device_resident_blob_decompress(oracle):
    """A blob in device memory is parsed through a sparse host mirror and read in place."""
    import torch

    a = S.smooth_noise((65, 40, 33), seed=9)
    blob = P.mgard_compress(a, 1e-3)
    d = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
    y = P.mgard_decompress(d).values
    assert np.array_equal(y.view(np.uint8), oracle.mgard_decompress(blob).view(np.uint8))
    bad = bytearray(blob)
    bad[len(blob) // 2] ^= 0x40
    want = oracle.mgard_decompress(bytes(bad))
    got = P.mgard_decompress(torch.from_numpy(np.frombuffer(bytes(bad), np.uint8).copy()).cuda()).values
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    with pytest.raises(CorruptStreamError):
        P.mgard_decompress(d[:60])


def test_pageable_staging_matches_pinned_and_device():
    """Plain numpy / bytes (pageable) go through the pinned staging rings: results must equal the
    pinned-host and device-resident paths byte for byte (sizes that leave partial 16 MB slots)."""
    torch = pytest.importorskip("torch")
    from paper_2503_06322_b200 import zfp as Z

    a = S.smooth_noise((301, 300, 203), seed=5)          # 73 MB fp32: 5 slots, a partial last one
    pin = torch.from_numpy(a.copy()).pin_memory()
    dev = torch.from_numpy(a).cuda()
    blob = P.mgard_compress(a, 1e-4)
    assert blob == P.mgard_compress(pin, 1e-4) == P.mgard_compress(dev, 1e-4)
    y = P.mgard_decompress(blob).values
    yp = torch.empty(a.shape, dtype=torch.float32).pin_memory()
    P.mgard_decompress(torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory().numpy(), out=yp.numpy())
    assert np.array_equal(y.view(np.uint32), yp.numpy().view(np.uint32))
    # a bytes slice at an odd offset (unaligned pageable source)
    buf = bytearray(b"\x00" * 3 + blob)
    y2 = P.mgard_decompress(memoryview(buf)[3:]).values
    assert np.array_equal(y.view(np.uint32), y2.view(np.uint32))
    z = Z.zfp_compress(a, 11)
    assert z == Z.zfp_compress(pin, 11)
    assert np.array_equal(Z.zfp_decompress(z).values.view(np.uint32),
                          Z.zfp_decompress(torch.from_numpy(np.frombuffer(z, np.uint8).copy()).cuda()).values.view(np.uint32))
