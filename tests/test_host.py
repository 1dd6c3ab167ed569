"""Host-side logic and the C ABI surface (CPU only; no kernel launches)."""
import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import _lib
from paper_2503_06322_b200 import synthetic as S
from paper_2503_06322_b200.huffman import FrequencyTable, build_codebook
from paper_2503_06322_b200.mgard import _abs_mapping

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hpdr_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hpdr_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_lib._SIGS), set(syms) - set(_lib._SIGS)


def test_library_is_sm100a_only():
    so = open(_lib.SO_PATH, "rb").read()
    assert b"sm_100a" in so or b"compute_100a" in so


def test_codebook_c_abi_matches_reference(huffman_golden, kat):
    meta, data = huffman_golden
    for j, d in enumerate(meta["codebooks"]):
        b = build_codebook(FrequencyTable(d, data[f"cbcounts{j}"]))
        assert np.array_equal(b.lengths, data[f"cblengths{j}"]), j
        assert np.array_equal(b.codes, data[f"cbcodes{j}"]), j
    for name, v in kat["codebook"].items():
        b = build_codebook(FrequencyTable(len(v["freq"]), np.array(v["freq"])))
        assert b.lengths.tolist() == v["lengths"] and b.codes.tolist() == v["codes"], name
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    with pytest.raises(P.ValidationError, match="exceeds 32"):
        build_codebook(FrequencyTable(40, np.array(fib)))
    with pytest.raises(P.ValidationError):
        build_codebook(FrequencyTable(3, np.zeros(3)))


def test_hierarchy_mirror(kat):
    for dims, h in kat["hierarchy"].items():
        dims = eval(dims)
        hh = P.build_hierarchy(dims)
        assert hh.total_levels == h["L"]
        assert [list(map(int, c)) for c in hh.level_counts] == h["counts"]
        assert list(map(int, hh.level_element_counts())) == h["owned"]
        assert hh.coarsest_flat_indices().tolist()[:64] == h["coarsest"]
        assert [list(map(int, m[-1])) for m in hh.index_maps] == h["maps_last"]
    with pytest.raises(P.ValidationError):
        P.build_hierarchy([3, 0])


def test_tensor_and_errors():
    with pytest.raises(P.ValidationError):
        P.TensorData((), P.DType.F32, np.zeros(0, np.float32))
    with pytest.raises(P.ValidationError):
        P.TensorData((1, 1, 1, 1, 1), P.DType.F32, np.zeros(1, np.float32))
    with pytest.raises(P.ValidationError):
        P.TensorData((2,), P.DType.F32, np.zeros(2, np.float64))
    t = P.TensorData.from_array(np.zeros((3, 4), np.float64))
    assert t.rank == 2 and t.dtype == P.DType.F64 and t.nbytes == 96
    assert issubclass(P.ValidationError, ValueError) and issubclass(P.ValidationError, P.HpdrError)
    e = P.CorruptStreamError("x", bit_offset=17)
    assert e.bit_offset == 17 and P.CorruptStreamError("y").bit_offset == -1
    assert P.DTYPE_CODES[P.DType.F32] == 0 and P.DTYPE_CODES[P.DType.U8] == 6


def test_abs_mapping_is_exact():
    for e in (1e-3, 0.5, 3.0, 1.0, 1024.0, 7e5, 2.0 ** -40):
        eb_rel, (lo, hi) = _abs_mapping(e)
        assert 0.0 < eb_rel < 1.0
        assert eb_rel * (hi - lo) == e


def test_context_key_digest_matches_reference_formula():
    k = P.ContextKey.make("mgard", (4, 5), "f32", eb_rel=1e-3, dict_size=4096)
    text = repr(("mgard", (4, 5), "f32", (("dict_size", 4096), ("eb_rel", 1e-3))))
    assert k.digest == int.from_bytes(hashlib.blake2b(text.encode(), digest_size=8).digest(), "little")


def test_product_fails_loudly_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(P.DeviceError):
        P.mgard_compress(np.zeros((4, 4), np.float32), 1e-3)


def test_synthetic_generators_are_pinned():
    cfg = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
    assert S.sha256(S.grf((129,) * 3, m=8, seed=0)) == cfg["C1_grf129_abs1e-3"]["input_sha"]
    assert S.sha256(S.nyx_like((129,) * 3, "temperature")) == cfg["C3_temperature_129_0.01"]["input_sha"]


def test_oracle_matches_reference_at_config_scale(oracle):
    cfg = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
    c = cfg["C1_grf129_abs1e-3"]
    blob = oracle.mgard_compress(S.grf((129,) * 3, m=8, seed=0), 1e-3, value_range=(0.0, 1.0))
    assert hashlib.sha256(blob).hexdigest() == c["blob_sha"]
    c = cfg["C3_velocity_x_129_1e-05"]   # 63% outliers, blob larger than the input
    blob = oracle.mgard_compress(S.nyx_like((129,) * 3, "velocity_x"), 1e-5)
    assert hashlib.sha256(blob).hexdigest() == c["blob_sha"]


def test_default_device_follows_process_placement(monkeypatch):
    """One process per GPU: a call without device= runs on the rank's GPU (HPDR_DEVICE, then
    torch's current device once CUDA is initialised, then LOCAL_RANK), or on a tensor's own."""
    from paper_2503_06322_b200 import _lib

    monkeypatch.delenv("HPDR_DEVICE", raising=False)
    monkeypatch.setenv("LOCAL_RANK", "3")
    assert _lib.default_device() in (3, 0) if _torch_cuda_initialized() else _lib.default_device() == 3
    monkeypatch.setenv("HPDR_DEVICE", "5")
    assert _lib.default_device() == 5

    class FakeDev:
        type, index = "cuda", 6

    class FakeTensor:
        device = FakeDev()

    assert _lib.default_device(FakeTensor()) == 6


def _torch_cuda_initialized():
    import sys

    t = sys.modules.get("torch")
    try:
        return bool(t is not None and t.cuda.is_initialized())
    except Exception:   # noqa: BLE001
        return False


def test_bytes_sink_trims_in_place_and_keeps_content():
    """The drop-in's result allocator (_lib.BytesSink): a size-hinted, pre-touched bytes object is
    trimmed to the exact blob size in place; a larger blob gets a fresh object; content is kept."""
    import ctypes as C

    from paper_2503_06322_b200 import _lib

    old = _lib.BytesSink.MIN_HINT
    _lib.BytesSink.MIN_HINT = 0
    try:
        for hint, n in ((4 << 20, 3 << 20), (1 << 20, 3 << 20), (0, 5000)):
            s = _lib.BytesSink(hint)
            p = s._alloc(None, n)
            C.memset(p, 0x5A, n)
            C.memset(p + n // 2, 0x33, 1)
            b = s.take()
            assert type(b) is bytes and len(b) == n
            assert b[0] == 0x5A and b[n - 1] == 0x5A and b[n // 2] == 0x33
    finally:
        _lib.BytesSink.MIN_HINT = old
